# The round-end tiers in one gpurun call: pytest -m gpu, smoke(), bench.py and a launch list.
#   bash tools/final_check.sh <tag>
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.txt 2>&1; echo "tests rc=$?" >> gpurun_out/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/status_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/status_$TAG.txt
