"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import io
import json
import sys


def shares(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for r in rows:
        if r.get("Metric Name", "gpu__time_duration.sum").startswith("dram__bytes"):
            name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
            if "at::" not in r["Kernel Name"] and "cub::" not in r["Kernel Name"]:
                v = float(r["Metric Value"].replace(",", ""))
                agg[name][2] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        if "at::" in r["Kernel Name"] or "cub::" in r["Kernel Name"]:  # torch kernels of the model / input construction
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ms = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
        agg[name][0] += ms
        agg[name][1] += 1
    tot = sum(a[0] for a in agg.values())
    out = sorted(((k, round(v[0], 3), v[1], round(v[0] / tot, 4), round(v[2] / 1e9, 3)) for k, v in agg.items()),
                 key=lambda x: -x[1])
    return tot, out


if __name__ == "__main__":
    tot, out = shares(sys.argv[1])
    print(f"total ms {tot:.2f}")
    for o in out:
        print(f"  {o[0]:28s} {o[1]:9.3f} ms  {o[2]:5d} launches  {100 * o[3]:5.1f}%  {o[4]:8.3f} GB DRAM")
    if len(sys.argv) > 2:
        json.dump({"total_ms": tot, "kernels": [dict(name=a, ms=b, launches=c, share=d, dram_gb=e) for a, b, c, d, e in out]},
                  open(sys.argv[2], "w"), indent=1)
