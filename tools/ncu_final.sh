mkdir -p gpurun_out
STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^attn_ps_kernel$' -s 16 -c 1 -o gpurun_out/ncu_r02c_rc_attn -f python tools/profile_step.py > gpurun_out/ncu_r02c_rc_attn.log 2>&1; echo "rc_attn rc=$?"
STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^s1_attn_tc_kernel$' -s 16 -c 1 -o gpurun_out/ncu_r02c_qp_attn -f python tools/profile_step.py > gpurun_out/ncu_r02c_qp_attn.log 2>&1; echo "qp_attn rc=$?"
STEPS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r02d.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?"
