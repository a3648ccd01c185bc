einsum: ij,kl,njl->nik
row: G1,G2,X
array: G1 float32 64x64
array: G2 float32 64x64
array: X float32 4096x64x64
