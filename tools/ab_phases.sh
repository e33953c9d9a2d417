# A/B of compile-time variants on one box: graph-replayed phase times, default lib vs
# PKV_LIB alternatives given as arguments (paper_2602_02579_b200/libpkv_*.so)
mkdir -p gpurun_out
for i in 1 2; do
  echo "default $(timeout 600 python tools/graph_phases.py 2>/dev/null | tail -1)" >> gpurun_out/ab_phases.txt
  for alt in "$@"; do
    echo "$alt $(PKV_LIB=$alt timeout 600 python tools/graph_phases.py 2>/dev/null | tail -1)" >> gpurun_out/ab_phases.txt
  done
done
