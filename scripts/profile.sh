#!/bin/bash
# Round profile capture (run under gpurun): launch list of one bench GCN step,
# launch list of one GAT layer step, of one Gat2 (config 4, 8x256) model step, and ncu --set full captures of the top
# kernels of both.  Outputs -> gpurun_out/, summarised by
# scripts/summarize_profiles.py into profiles/<tag>/.
set -x
TAG=${1:-r1}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-model-cpu --no-large --no-parity > gpurun_out/launches_${TAG}.log 2>&1
ONE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_|gemm|split" --csv --log-file gpurun_out/gat_launches_${TAG}.csv \
    python scripts/kbench.py gat > gpurun_out/gat_launches_${TAG}.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_|gemm|split" --csv --log-file gpurun_out/gat2_launches_${TAG}.csv \
    python scripts/dev/gat2_step.py 256 > gpurun_out/gat2_launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_lean|k_gemm_tc|k_colsum" \
    -s 12 -c 6 -o gpurun_out/full_${TAG} \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-model-cpu --no-large --no-parity > gpurun_out/full_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_gat_attnagg|k_gat_attn4|k_gat_agg2|k_gat_sddmm|k_gat_sbwd4|k_gat_col2|k_node_scores" \
    -s 6 -c 6 -o gpurun_out/full_gat_${TAG} \
    python scripts/kbench.py gat > gpurun_out/full_gat_${TAG}.log 2>&1
# the GAT primitives bench.py times standalone (sddmm2, perm-indirect col2)
ncu --set full --clock-control none --import-source on -k regex:"k_gat_sddmm2|k_gat_col2" \
    -s 2 -c 2 -o gpurun_out/full_prims_${TAG} \
    python scripts/dev/gat_prims.py > gpurun_out/full_prims_${TAG}.log 2>&1
ls -la gpurun_out
