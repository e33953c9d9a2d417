mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "probe or cacheblend or kvshare" --timeout 600 > gpurun_out/gpu_tests_probe.txt 2>&1; echo probe rc=$?; tail -2 gpurun_out/gpu_tests_probe.txt
for lib in default base; do
  if [ $lib = base ]; then export PKV_LIB=paper_2602_02579_b200/libpkv_base.so; fi
  STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:s1_ --csv --log-file gpurun_out/s1_$lib.csv python tools/profile_step.py > /dev/null 2>&1
  python - <<PY
import csv,io,collections
t=open("gpurun_out/s1_$lib.csv").read().splitlines()
st=next(i for i,l in enumerate(t) if l.startswith('"ID"'))
r=list(csv.DictReader(io.StringIO("\n".join(t[st:]))))
a=collections.defaultdict(list)
for x in r: a[x["Kernel Name"].split("(")[0][:40]].append(float(x["Metric Value"].replace(",",""))/1e3)
for k,v in a.items(): print("$lib", k, len(v), round(sum(v)/len(v),1), "us avg", round(sum(v),1), "us total")
PY
done
