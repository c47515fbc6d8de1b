for shape in "8 32" "8 64" "8 256"; do for r in 1 2; do
  SGNN_GAT_WIDE_R=$r ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_gat" python scripts/dev/gat_layer.py $shape > "gpurun_out/lay1_${shape// /x}_$r.csv" 2>/dev/null
done; done
