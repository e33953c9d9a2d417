"""Per-kernel SASS evidence of the tcgen05 / TMA datapath in the built libpkv.so.

    python tools/sass_summary.py [out.json]

Counts, per kernel (demangled), the Blackwell instructions that prove the design:
UTCHMMA / UTCQMMA (tcgen05.mma, `.2CTA` = cta_group::2), LDTM / STTM (tcgen05.ld/st),
UTMALDG (TMA tensor loads), UBLKCP (bulk copies), MUFU.EX2, and the register count.
"""
import collections
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "paper_2602_02579_b200" / "libpkv.so"
PAT = re.compile(r"\b(UTC[A-Z]*MMA(?:\.2CTA)?|LDTM|STTM|UTMALDG|UTMASTG|UBLKCP|MUFU\.EX2|UTCBAR(?:\.2CTA)?)")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for tok in PAT.findall(line):
            counts[cur][tok] += 1
    res = subprocess.run(["cuobjdump", "-res-usage", str(SO)], capture_output=True, text=True).stdout
    regs = {}
    for fn, r in re.findall(r"Function (\S+):\s*\n\s*REG:(\d+)", res):
        regs[fn] = int(r)
    dm = demangle(list(counts))
    kernels = {dm[k]: dict(sorted(v.items()), regs=regs.get(k)) for k, v in counts.items() if v}
    total = collections.Counter()
    for v in counts.values():
        total.update(v)
    out = {"library": str(SO.relative_to(ROOT)), "arch": "sm_100a", "totals": dict(sorted(total.items())),
           "kernels": kernels}
    path = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r02" / "sass_summary.json"
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out["totals"]))


if __name__ == "__main__":
    main()
