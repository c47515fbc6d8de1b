0 1 abc
1 2
