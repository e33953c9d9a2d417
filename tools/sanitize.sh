# compute-sanitizer over smoke() (one small prefill through every default kernel) and the
# kernel unit tests.  synccheck is not run: it flags mbarrier phases that complete without a
# waiter (pv_full / kv_empty by design: the consumers wait on later phases, ordered by s_full).
mkdir -p gpurun_out
CS="/usr/local/cuda/bin/compute-sanitizer --print-limit 20"
SMOKE='import __graft_entry__ as g; g.smoke(); print("smoke ok")'
timeout 1200 $CS --tool memcheck python -c "$SMOKE" > gpurun_out/sanitize_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.txt
timeout 1200 $CS --tool racecheck python -c "$SMOKE" > gpurun_out/sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.txt
timeout 1800 $CS --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_gpu_kernels.py -k "not opt_in" > gpurun_out/sanitize_kernels.txt 2>&1; echo "kernels memcheck rc=$?" >> gpurun_out/sanitize_kernels.txt
# head dim 128 (the default persistent attention, the tcgen05 narrow pass, CTA-pair GEMMs) at
# Llama width, the fused finalize, and the sharded / token-parallel paths
timeout 2400 $CS --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "llama_width or mistral_width" > gpurun_out/sanitize_parity128.txt 2>&1; echo "parity128 memcheck rc=$?" >> gpurun_out/sanitize_parity128.txt
timeout 2400 $CS --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_gpu_tp.py > gpurun_out/sanitize_tp.txt 2>&1; echo "tp memcheck rc=$?" >> gpurun_out/sanitize_tp.txt
timeout 2400 $CS --tool racecheck python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "prophet_slice and llama_width" > gpurun_out/sanitize_race128.txt 2>&1; echo "race128 rc=$?" >> gpurun_out/sanitize_race128.txt
timeout 1200 $CS --tool initcheck python -c "$SMOKE" > gpurun_out/sanitize_initcheck.txt 2>&1; echo "initcheck rc=$?" >> gpurun_out/sanitize_initcheck.txt
for t in test_gpu_api test_gpu_decode test_gpu_prefill test_gpu_chunkfile test_gpu_acceptance; do
  timeout 1500 $CS --tool memcheck python -m pytest -q -p no:cacheprovider tests/$t.py > gpurun_out/sanitize_$t.txt 2>&1; echo "$t rc=$?" >> gpurun_out/sanitize_$t.txt
done
