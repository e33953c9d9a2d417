mkdir -p gpurun_out
export STEPS=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_s1.csv python tools/profile_step.py > gpurun_out/launches_s1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:s1_score_tc_kernel -s 8 -c 1 -o gpurun_out/ncu_s1score -f python tools/profile_step.py > gpurun_out/ncu_s1score.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:s1_attn_tc_kernel -s 8 -c 1 -o gpurun_out/ncu_s1attn -f python tools/profile_step.py > gpurun_out/ncu_s1attn.log 2>&1
