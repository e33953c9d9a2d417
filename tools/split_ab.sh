# Correctness + A/B of the split-S persistent attention (PKV_ATTN_SPLIT_S=1).
mkdir -p gpurun_out
PKV_ATTN_SPLIT_S=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "attn or attention" > gpurun_out/split_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/split_tests.txt
for i in 1 2 3; do
  for setting in "PKV_ATTN_SPLIT_S=0" "PKV_ATTN_SPLIT_S=1"; do
    echo "[$setting] attn $(env $setting timeout 300 python tools/bench_attn.py 2>/dev/null | tail -1)" >> gpurun_out/split_ab.txt
  done
done
for i in 1 2; do
  for setting in "PKV_ATTN_SPLIT_S=0" "PKV_ATTN_SPLIT_S=1"; do
    echo "[$setting] ttft $(env $setting timeout 600 python tools/graph_ttft.py 5 2>/dev/null | tail -1)" >> gpurun_out/split_ab.txt
  done
done
