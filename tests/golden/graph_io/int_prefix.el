12abc 3
