cd $GRAFT_REPO_ROOT
ONE=1 SGNN_GEMM_EXP=86 ncu --set full --clock-control none -k regex:"k_gemm_tc" -s 2 -c 1 -o gpurun_out/gemm_exp86 python scripts/kbench.py nn > /dev/null 2>&1
