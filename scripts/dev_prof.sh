cd $GRAFT_REPO_ROOT
ONE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none --csv -k regex:"k_gat|k_node|k_gemm|k_split|k_col|k_reduce|k_attgrad" python scripts/kbench.py gat > gpurun_out/gat_launch.csv 2>/dev/null
