source target
0 1
1 2
