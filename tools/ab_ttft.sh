# A/B of library builds / env knobs on one box: graph-replayed TTFT and phase split, and
# the Stage-II GEMM shapes, each setting in its own process (knobs are read once).
#   bash tools/ab_ttft.sh "ENV=.. ENV2=.." "PKV_LIB=paper_2602_02579_b200/libpkv_base.so" ...
mkdir -p gpurun_out
for i in 1 2; do
  for setting in "" "$@"; do
    echo "[$setting] ttft $(env $setting timeout 600 python tools/graph_ttft.py 5 2>/dev/null | tail -1)" >> gpurun_out/ab_ttft.txt
    echo "[$setting] phases $(env $setting timeout 600 python tools/graph_phases.py 2>/dev/null | tail -1)" >> gpurun_out/ab_ttft.txt
  done
done
for setting in "" "$@"; do
  echo "[$setting] gemm $(env $setting EPI=2 timeout 600 python tools/bench_stage2_gemm.py 2>/dev/null | tail -1)" >> gpurun_out/ab_ttft.txt
done
