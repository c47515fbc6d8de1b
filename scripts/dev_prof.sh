cd $GRAFT_REPO_ROOT
ONE=1 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc" -s 2 -c 1 -o gpurun_out/gemm_nn python scripts/kbench.py nn > /dev/null 2>&1
