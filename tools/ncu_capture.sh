#!/bin/bash
# ncu evidence for the top kernels of one prefill step (run under gpurun, 1 GPU).
#   bash tools/ncu_capture.sh [tag]
# -> gpurun_out/ncu_<tag>_<kernel>.ncu-rep (+ a launch list of one step)
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
export STEPS=1
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name, name-base, regex, skip
  timeout 900 $NCU --kernel-name-base $2 -k "regex:$3" -s $4 -c 1 -o $OUT/ncu_${TAG}_$1 -f \
    python tools/profile_step.py > $OUT/ncu_${TAG}_$1.log 2>&1
  echo "$1 rc=$?" >> $OUT/ncu_${TAG}.status
}
cap rc_attn function '^attn_ps_kernel$' 16
cap rc_gate_up demangled 'gemm_tc_kernel<\(int\)256, \(int\)3,' 16
cap rc_down demangled 'gemm_tc_kernel<\(int\)256, \(int\)2,' 33
cap rc_o demangled 'gemm_tc_kernel<\(int\)256, \(int\)2,' 32
cap rc_qkv demangled 'gemm_tc_kernel<\(int\)256, \(int\)4,' 16
cap qp_attn function '^s1_attn_tc_kernel$' 16
cap qp_score function '^s1_score_tc_kernel$' 16
cap qp_proj demangled 'gemm_tc_kernel<\(int\)96, \(int\)5,' 40
cap assemble function '^assemble_kernel$' 0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_${TAG}.csv python tools/profile_step.py > $OUT/launches_${TAG}.log 2>&1
echo "launches rc=$?" >> $OUT/ncu_${TAG}.status
