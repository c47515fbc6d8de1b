#!/bin/bash
# Round profile capture (run under gpurun): launch list of one bench step and
# ncu --set full captures of the step's top kernels.  Outputs -> gpurun_out/.
set -x
TAG=${1:-r1}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_lean|k_gemm_tc|k_colsum" \
    -s 12 -c 6 -o gpurun_out/full_${TAG} \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gat_fwd_fast|k_gat_bwd_row_fast|k_gat_bwd_col_fast" \
    -s 3 -c 3 -o gpurun_out/full_gat_${TAG} \
    python scripts/kbench.py gat > gpurun_out/full_gat_${TAG}.log 2>&1
ls -la gpurun_out
