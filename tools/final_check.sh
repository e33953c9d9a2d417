mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02t.txt 2>&1; echo "tests rc=$?" >> gpurun_out/status_r02t.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02t.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/status_r02t.txt
timeout 900 python bench.py > gpurun_out/bench_r02t.json 2> gpurun_out/bench_r02t.err; echo "bench rc=$?" >> gpurun_out/status_r02t.txt
STEPS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r02e.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?" >> gpurun_out/status_r02t.txt
