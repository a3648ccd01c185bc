einsum: xre,xij,ej->rei
row: J,D,u1
row: J,D,u2
row: J,D,u3
array: D float32 3x10x10
array: J float32 3x3x2000000
array: u1 float32 2000000x10
array: u2 float32 2000000x10
array: u3 float32 2000000x10
