# Stage-II attention A/B on one box: isolated graph timing of the row kernel (default)
# against the two-warps-per-row kernel, then the pipeline phases
mkdir -p gpurun_out
for i in 1 2; do
  echo "row $(timeout 300 python tools/bench_attn.py 2>/dev/null | tail -1)" >> gpurun_out/attn_ab.txt
  echo "old $(PKV_ATTN_ROW=0 timeout 300 python tools/bench_attn.py 2>/dev/null | tail -1)" >> gpurun_out/attn_ab.txt
done
for pp in 0 2 3; do
  echo "row rpoly=$pp $(PKV_ATTN_RPOLY=$pp timeout 300 python tools/bench_attn.py 2>/dev/null | tail -1)" >> gpurun_out/attn_ab.txt
done
echo "phases $(timeout 600 python tools/graph_phases.py 2>/dev/null | tail -1)" >> gpurun_out/attn_ab.txt
