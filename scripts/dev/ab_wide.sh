for shape in "8 64" "8 128" "4 128" "8 256"; do for r in 2 4 8; do
  SGNN_GAT_WIDE_R=$r ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_gat" python scripts/dev/gat_layer.py $shape > "gpurun_out/lay_${shape// /x}_$r.csv" 2>/dev/null
done; done
