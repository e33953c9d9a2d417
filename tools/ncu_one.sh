# ncu --set full of one launch of kernel regex $1 (skip $2 launches) in tools/profile_step.py
# -> gpurun_out/ncu_$3.ncu-rep
mkdir -p gpurun_out
STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${2:-8} -c 1 \
  -o gpurun_out/ncu_$3 -f python tools/profile_step.py > gpurun_out/ncu_$3.log 2>&1
