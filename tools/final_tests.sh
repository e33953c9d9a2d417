# The round-end GPU tiers in one call: pytest -m gpu and smoke() (outputs under gpurun_out/).
#   bash tools/final_tests.sh <tag>
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.txt 2>&1; echo "tests rc=$?" >> gpurun_out/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/status_$TAG.txt
