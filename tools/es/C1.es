einsum: xre,xij,ej->rei
row: J,D,u1
row: J,D,u2
row: J,D,u3
array: D float64 3x10x10
array: J float64 3x3x10000
array: u1 float64 10000x10
array: u2 float64 10000x10
array: u3 float64 10000x10
