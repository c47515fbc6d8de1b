# a comment

0 1 # trailing comment
   
1 0 3
