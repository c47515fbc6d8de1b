0 1 1.0 extra
