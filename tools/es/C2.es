einsum: xai,xbm,xcn,xyeabc,yaj,ybk,ycl,ejkl->eimn
row: A1,A2,A3,G,A1,A2,A3,u1
row: A1,A2,A3,G,A1,A2,A3,u2
row: A1,A2,A3,G,A1,A2,A3,u3
row: A1,A2,A3,G,A1,A2,A3,u4
row: A1,A2,A3,G,A1,A2,A3,u5
row: A1,A2,A3,G,A1,A2,A3,u6
row: A1,A2,A3,G,A1,A2,A3,u7
row: A1,A2,A3,G,A1,A2,A3,u8
array: A1 float64 3x5x5
array: A2 float64 3x5x5
array: A3 float64 3x5x5
array: G float64 3x3x2000000x5x5x5
array: u1 float64 2000000x5x5x5
array: u2 float64 2000000x5x5x5
array: u3 float64 2000000x5x5x5
array: u4 float64 2000000x5x5x5
array: u5 float64 2000000x5x5x5
array: u6 float64 2000000x5x5x5
array: u7 float64 2000000x5x5x5
array: u8 float64 2000000x5x5x5
