einsum: ij,kl,njl->nik
row: G1,G2,X
array: G1 float64 64x64
array: G2 float64 64x64
array: X float64 4096x64x64
