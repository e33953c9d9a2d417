"""ProphetKV selective-recompute prefill benchmark (BASELINE.json metric).

Step = one full prefill of one RAG request: assemble 16 precomputed 2048-token
chunks (Llama-3-8B shape, random init, synthetic inputs) into the paged cache,
score the context with the 32-token query (fp32-faithful narrow pass), fuse +
top-k at p = 0.2, Stage-II recompute of k = 6554 tokens, finalize -> first-token
logits.

Inputs: SYN1 (paper_2602_02579_b200/synthetic.py) -- random-init weights at the reference's
init scale, chunk K/V and query generated on the device and reproduced bit for bit by the
CPU oracle; the run is checked in place against tests/golden/anchor_c3.npz ("parity").

Multi-GPU (one process per GPU; `--gpus N` starts torchrun itself when WORLD_SIZE is unset), --mode:
  heads     (default for N > 1; BASELINE configs[2]) one 32k request head-sharded over
            the N GPUs (tensor parallel, paper_2602_02579_b200.tp): per-layer NCCL sums of
            the per-token score partials before the global top-k and of the o/down
            projection outputs; value = s / TTFT (strong scaling)
  tokens    one 32k request: every GPU holds the full model and cache; the scoring pass is
            head-sharded over each GPU's head slice (per-layer score all-reduce), Stage II
            repairs each GPU's share of the selected rows and all-gathers the fresh cache
            entries per layer (DeviceModel.rows); value = s / TTFT (strong scaling)
  requests  (configs[4]-style) one independent request per GPU, no data-path
            collective; value = N * s / TTFT (weak scaling)

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode heads|tokens|requests]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[2]: Llama-3-8B shape, 32k context of 16 chunks, 20% recompute
    "llama3-8b-32k": dict(n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, hidden_dim=4096, ffn_dim=14336,
                          vocab_size=128256, rope_theta=500000.0, n_chunks=16, chunk_len=2048),
    # configs[1]: Mistral-7B shape, 8k context of 8 chunks
    "mistral-7b-8k": dict(n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, hidden_dim=4096, ffn_dim=14336,
                          vocab_size=32000, rope_theta=1000000.0, n_chunks=8, chunk_len=1024),
    # configs[4]: Llama-3-8B shape, 128k context of 64 chunks, one request per GPU (--mode requests)
    "llama3-8b-128k": dict(n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, hidden_dim=4096, ffn_dim=14336,
                           vocab_size=128256, rope_theta=500000.0, n_chunks=64, chunk_len=2048),
}
def metric_name(cfgd: dict, p: float) -> str:
    s = cfgd["n_chunks"] * cfgd["chunk_len"]
    return f"effective prefill tok/s @{s // 1024}k ctx, {p * 100:g}% recompute (TTFT = s / value)"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return float("nan")
        sm = [num(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": num(rows[0][1]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(num(r[2]) for r in rows)}


# --------------------------------------------------------------------- CPU baseline
def cpu_sample(cfgd: dict, p: float, m: int = 32, n_rows: int = 256, seed: int = 0):
    """Time the reference algorithm (oracle port of pikv) on a bounded sample of the
    workload and extrapolate to the full request: one layer of the full-width model
    at the full context s; Stage II on n_rows of the k selected rows (its cost is
    linear in rows: dense k x s attention per the reference); x n_layers."""
    from oracle import pikv_oracle as O
    L = cfgd["n_layers"]
    c1 = O.Cfg(1, cfgd["n_heads"], cfgd["n_kv_heads"], cfgd["head_dim"], cfgd["hidden_dim"], cfgd["ffn_dim"],
               cfgd["vocab_size"], cfgd["rope_theta"])
    rng = np.random.default_rng(seed)
    D, F, V, KV = c1.hidden_dim, c1.ffn_dim, c1.vocab_size, c1.kv_dim
    HQ = c1.n_heads * c1.head_dim

    def mat(a, b):
        return (rng.standard_normal((a, b), dtype=np.float32) / np.float32(math.sqrt(a)))

    w = O.Weights(embed=rng.standard_normal((V, D), dtype=np.float32),
                  layers=[O.Layer(np.ones(D, np.float32), mat(D, HQ), mat(D, KV), mat(D, KV), mat(HQ, D),
                                  np.ones(D, np.float32), mat(D, F), mat(D, F), mat(F, D))],
                  final_norm=np.ones(D, np.float32), lm_head=mat(D, V), _fp="cpu-sample")
    chunks = []
    for ci in range(cfgd["n_chunks"]):
        t = cfgd["chunk_len"]
        kn = [O.bf16_round(rng.standard_normal((t, c1.n_kv_heads, c1.head_dim), dtype=np.float32))]
        vv = [O.bf16_round(rng.standard_normal((t, c1.n_kv_heads, c1.head_dim), dtype=np.float32))]
        chunks.append(O.Chunk(ci, "cpu-sample", rng.integers(0, V, t), kn, vv))
    query = rng.integers(0, V, m).tolist()
    tm = {}
    t0 = time.perf_counter()
    cache = O.stitch(chunks, c1)
    tm["assemble"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    per, fused = O.prophet_scores(w, c1, cache, query)
    tm["score"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.logits_of(w, c1, np.zeros((m, D), np.float32) + 0.01, None)
    tm["head"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sel, k = O.select(fused, p)
    tm["select"] = time.perf_counter() - t0
    sample = sel[:: max(1, len(sel) // n_rows)][:n_rows]
    t0 = time.perf_counter()
    O.repair(w, c1, cache, sample)
    tm["repair_sample"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.finalize(w, c1, cache, query)
    tm["finalize"] = time.perf_counter() - t0
    body = tm["assemble"] + (tm["score"] - tm["head"]) + (tm["finalize"] - tm["head"])
    ttft = L * body + 2 * tm["head"] + tm["select"] + L * tm["repair_sample"] * (k / len(sample))
    return ttft, tm, k, len(sample), sum(tm.values())


def full_anchor_run(args):
    """The one FULL CPU run of this workload: the layer-streamed oracle over all 32 layers
    and all k rows that produced tests/golden/anchor_c3.npz (tests/golden/make_anchor.py,
    8 threads of the build container, not this box) -- the check on the extrapolation."""
    path = ROOT / "tests" / "golden" / "anchor_c3.npz"
    if args.config != "llama3-8b-32k" or not path.exists():
        return None
    meta = json.loads(str(np.load(path)["meta"]))
    return {"wall_s": meta["cpu_seconds"], "threads": 8, "where": "build container (8 cores)",
            "what": "oracle/anchor.py: assemble + score_prophet + select + recompute (all k rows, "
                    "causal-visible attention per row block) + finalize, L = 32, s = 32768"}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def cpu_threads():
    """Host threading of the CPU baseline: cores in the affinity mask, OMP / BLAS threads."""
    info = {"affinity_cores": cpu_cores(), "os_cpu_count": os.cpu_count(),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:  # noqa: BLE001 -- informational
        pass
    return info


def arm_config(args, cfgd, world, heads, tokens=False):
    """The `config` dict of a bench line -- identical for our arm and the reference arm."""
    s = cfgd["n_chunks"] * cfgd["chunk_len"]
    return {"workload": args.config, "model": "Llama-3-8B shape" if "llama" in args.config else "Mistral-7B shape",
            "s": s, "chunks": cfgd["n_chunks"], "chunk_len": cfgd["chunk_len"], "m": args.m, "p": args.p,
            "k": math.ceil(args.p * s),
            "parallelism": (f"tp{world} (KV-head sharded, NCCL)" if heads else
                            f"tokens{world} (scoring KV-head sharded, Stage II token-parallel, NCCL)"
                            if tokens else f"request-dp{world}"),
            "inputs": f"SYN1 seed 0 (weights, chunk store, query: paper_2602_02579_b200/synthetic.py)"
            if args.chunks == "synthetic" else "SYN1 weights; chunk K/V precomputed on the GPU",
            "l2": "inputs larger than L2 (16 GB weights, 4.3 GB KV)"}


def ttft_floor_ms(cfgd, p, m, hbm_gbs, tflops):
    """Algorithmic TTFT floor: assembly + Stage-I weight streaming + final
    pass (HBM) + Stage-II GEMMs and causal-visible attention (tensor) at the peaks."""
    L, H, Hkv, dk, D, F, V = (cfgd[k] for k in ("n_layers", "n_heads", "n_kv_heads", "head_dim", "hidden_dim",
                                                 "ffn_dim", "vocab_size"))
    s = cfgd["n_chunks"] * cfgd["chunk_len"]
    k = math.ceil(p * s)
    params = L * (D * (H * dk + 2 * Hkv * dk) + H * dk * D + 3 * D * F)
    hbm = (4 * L * s * Hkv * dk * 2 + 2 * params * 2 + D * V * 2 + 2 * L * s * Hkv * dk * 2) / (hbm_gbs * 1e9)
    flops = 2.0 * k * params + 4.0 * L * H * dk * (k * (s + 1) / 2)
    return (hbm + flops / (tflops * 1e12)) * 1e3


def load_anchor(args, heads):
    """The oracle fixture of this exact workload (tests/golden/make_anchor.py), if any."""
    if args.config != "llama3-8b-32k" or args.chunks != "synthetic" or args.m != 32 or abs(args.p - 0.2) > 1e-12:
        return None
    path = ROOT / "tests" / "golden" / "anchor_c3.npz"
    if not path.exists():
        return None
    z = np.load(path)
    return json.loads(str(z["meta"])), {k: z[k] for k in z.files if k != "meta"}


def anchor_parity(pipe, anchor, heads):
    """In-run parity of the benchmarked request against the CPU oracle (north-star
    tolerances): per-layer scores, selection (tie band 1e-4), first-token logits and, when
    the selection is the reference's, the recomputed fp16 cache entries at 16 rows x L."""
    meta, z = anchor
    per = pipe.per_layer.cpu().numpy()
    k = int(meta["k"])
    sel = pipe.idx[:k].cpu().numpy().astype(np.int64)
    rel = float((np.abs(per - z["per_layer"]) / np.maximum(np.abs(z["per_layer"]), 1e-30)).max())
    fused = z["fused"]
    kth = np.sort(fused)[::-1][k - 1]
    band = np.abs(fused - kth) <= 1e-4 * abs(kth)
    a, b = set(sel.tolist()), set(z["sel"].tolist())
    sel_ok = len(a) == k and {i for i in a if not band[i]} == {i for i in b if not band[i]}
    lg = pipe.logits.cpu().numpy().astype(np.float64)
    lr = z["first_logits"].astype(np.float64)
    cos = float(lg @ lr / (np.linalg.norm(lg) * np.linalg.norm(lr)))
    out = {"fixture": "tests/golden/anchor_c3.npz (oracle on the same SYN1 inputs)", "per_layer_max_rel": rel,
           "tie_band": int(band.sum()), "sel_symdiff": len(a ^ b), "sel_ok": bool(sel_ok),
           "logits_max_abs": float(np.abs(lg - lr).max()), "logits_cos": cos}
    ok = rel <= 1e-4 and sel_ok and out["logits_max_abs"] <= 2e-2 and cos >= 0.999
    if not heads and a == b:
        cache, dk = pipe.cache, pipe.cfg.head_dim
        ix = z["sel"][z["kv_rows"]]
        err, kcos = 0.0, 1.0
        for li in range(pipe.cfg.n_layers):
            for pool, ref in ((cache.k_pool, z["kv_k"][li]), (cache.v_pool, z["kv_v"][li])):
                got = pool[li, :, ix, :dk].permute(1, 0, 2).float().cpu().numpy().astype(np.float64)
                err = max(err, float(np.abs(got - ref).max()))
                kcos = min(kcos, float((got.ravel() @ ref.ravel()) / (np.linalg.norm(got) * np.linalg.norm(ref))))
        out.update(kv_fp16_cache_max_abs=err, kv_min_cos=kcos, kv_rows=f"{len(ix)} selected rows x every layer")
        ok = ok and err <= 2e-2 and kcos >= 0.999
    out["pass"] = bool(ok)
    return out


def nccl_summary(path):
    """NCCL version / NVLS lines from the NCCL_DEBUG=INFO log of this rank."""
    try:
        lines = Path(path).read_text(errors="replace").splitlines()
    except OSError:
        return None
    pick = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if "NCCL INFO" in ln and
            any(t in ln for t in ("NCCL version", "NVLS", "nvls", "Channel 00", "comm 0x", "Init COMPLETE"))]
    return {"log": str(path), "nvls": any("NVLS" in ln and "enabled" in ln.lower() for ln in lines),
            "lines": pick[:12]}


def relaunch_under_torchrun(n):
    """`bench.py --gpus N` without a torchrun environment: start N ranks on this node."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} requested but {have} CUDA device(s) visible"}), flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd))


# ----------------------------------------------------------------------------- main
def run_reference(args, cfgd, rank, world):
    if rank != 0:
        return
    s = cfgd["n_chunks"] * cfgd["chunk_len"]
    times = []
    for i in range(args.warmup + args.steps):
        ttft, tm, k, n_s, wall = cpu_sample(cfgd, args.p, n_rows=args.ref_rows, seed=i)
        if i >= args.warmup:
            times.append(ttft)
    ttft = float(np.mean(times))
    value = s / ttft
    cores = cpu_cores()
    mode = args.mode if args.mode != "auto" else ("heads" if world > 1 else "requests")
    line = {"impl": "reference", "metric": metric_name(cfgd, args.p), "value": value, "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ttft * 1e3, "ttft_ms": ttft * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 accumulate)",
            "data": "synthetic", "config": arm_config(args, cfgd, world, mode == "heads" and world > 1,
                                                      mode == "tokens" and world > 1),
            "cpu_baseline": {"value": value, "unit": "tok/s", "cores": cores, "kind": "port", "threads": cpu_threads(),
                             "sample": f"oracle port of pikv, 1 layer at full width and s={s}, Stage II on {n_s} "
                                       f"of k={k} rows, extrapolated x{cfgd['n_layers']} layers and k/{n_s} rows; "
                                       f"phase seconds {json.dumps({a: round(b, 3) for a, b in tm.items()})}",
                             "full_run": full_anchor_run(args)},
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3-8b-32k", choices=list(CONFIGS))
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--full-steps", type=int, default=1, help="full-prefill comparator runs (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=128)
    ap.add_argument("--mode", default="auto", choices=["auto", "heads", "tokens", "requests"])
    ap.add_argument("--p-sweep", default="0.05,0.1,0.2,0.4", help="recompute ratios of the sweep ('' = skip)")
    ap.add_argument("--sweep-steps", type=int, default=3)
    ap.add_argument("--chunks", default="synthetic", choices=["synthetic", "precompute"])
    args = ap.parse_args()
    cfgd = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        relaunch_under_torchrun(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfgd, rank, world)
        return
    if world != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: reporting the {world} launched ranks",
              file=sys.stderr, flush=True)

    mode = args.mode if args.mode != "auto" else ("heads" if world > 1 else "requests")
    heads = mode == "heads" and world > 1
    tokens = mode == "tokens" and world > 1
    shared = heads or tokens  # one request over all ranks (strong scaling)
    nccl_log = None
    if shared:  # NCCL init / NVLS lines of this rank (summarised in the JSON line)
        out_dir = ROOT / "gpurun_out" if (ROOT / "gpurun_out").is_dir() else Path("/tmp")
        nccl_log = out_dir / f"nccl_rank{rank}.log"
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS,GRAPH")
        os.environ.setdefault("NCCL_DEBUG_FILE", str(nccl_log))

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    __graft_entry__.build()
    import paper_2602_02579_b200 as P
    from paper_2602_02579_b200 import _lib
    from paper_2602_02579_b200 import synthetic as S
    from paper_2602_02579_b200.pipeline import PrefillPipeline

    cfg = P.ModelConfig(**{k: cfgd[k] for k in ("n_layers", "n_heads", "n_kv_heads", "head_dim", "hidden_dim",
                                                "ffn_dim", "vocab_size", "rope_theta")})
    s = cfgd["n_chunks"] * cfgd["chunk_len"]

    def make_chunks(model, seed):
        """The request's chunk store: SYN1 keys/values (the inputs the oracle fixture was
        computed on), or precomputed on the GPU from SYN1 token ids (--chunks precompute)."""
        if args.chunks == "synthetic":
            return S.chunks(cfg, cfgd["n_chunks"], cfgd["chunk_len"], seed, model.fingerprint)
        from paper_2602_02579_b200.prefill import precompute_chunks_device
        toks = [S.token_ids(cfgd["chunk_len"], cfg.vocab_size, seed, S.tid_tokens(c)).cpu().numpy()
                for c in range(cfgd["n_chunks"])]
        out = precompute_chunks_device(model, cfg, toks)
        torch.cuda.synchronize()
        return out

    if heads:
        # one request, KV heads (and ffn blocks) sharded over the ranks; every rank builds
        # the same SYN1 model / chunk store and keeps its slice.  No fallback: a failing
        # communicator ends the run.
        from paper_2602_02579_b200 import tp
        comm = tp.nccl_comm()
        full = P.DeviceModel.synthetic(cfg, seed=0)
        full_chunks = make_chunks(full, 0)
        dm = full.shard(rank, world, comm.handle)
        del full
        chunks = tp.shard_chunks(full_chunks, rank, world)
        del full_chunks
        torch.cuda.empty_cache()
        qseed = 0
    elif tokens:
        # one request: every rank holds the full SYN1 model and chunk store, scores the whole
        # request (replicated, deterministic -> identical selections) and repairs its share of
        # the selected rows (DeviceModel.rows, pkv_recompute_rows)
        from paper_2602_02579_b200 import tp
        comm = tp.nccl_comm()
        full = P.DeviceModel.synthetic(cfg, seed=0)
        chunks = make_chunks(full, 0)
        dm = full.rows(comm)
        # the scoring pass head-sharded over this rank's head slice of the full cache
        stage1_dm = full.shard(rank, world, comm.handle)
        qseed = 0
    else:
        dm = P.DeviceModel.synthetic(cfg, seed=0)
        chunks = make_chunks(dm, rank)  # request r of the batch: chunk store / query seed r
        qseed = rank
    pipe = PrefillPipeline(dm, chunks, args.m, args.p, stage1_dm=stage1_dm if tokens else None)
    query = S.query(cfg, args.m, qseed)
    pipe.set_query(query)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        pipe.step()
    torch.cuda.synchronize()
    # eager steps with the native timers (CUDA events on the launching stream around each
    # kernel group): per-kernel device times for the roofline; counts our launches.  The
    # final pass runs serially here: overlapped with Stage II (the timed graph) its timer
    # scopes would include the per-layer waits and the time shared with Stage II kernels.
    overlap = pipe.final_overlap
    pipe.final_overlap = False
    _lib.timing(True)
    n0 = _lib.launch_count()
    for _ in range(args.steps):
        pipe.step()
    torch.cuda.synchronize()
    launches_per_step = (_lib.launch_count() - n0) // args.steps
    phases = _lib.timing_collect()
    _lib.timing(False)
    pipe.final_overlap = overlap
    eager_phases = {n: (v[0] / args.steps, v[1]) for n, v in phases.items()}
    phases = {n: (v[0] / args.steps, v[1] / args.steps) for n, v in phases.items()}
    # CUDA graph of one step for the timed region (eager launches if capture fails,
    # e.g. a collective back end that cannot be captured)
    launch_mode = "CUDA graph of one prefill step, replayed K times"
    try:
        pipe.capture()
        for _ in range(max(1, args.warmup)):
            pipe.replay()
    except Exception as e:  # noqa: BLE001
        launch_mode = f"eager launches (graph capture failed: {type(e).__name__})"
        pipe.replay = pipe.step
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(max(1, args.warmup)):
            pipe.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        pipe.replay()
    ev1.record(stream)
    torch.cuda.synchronize()
    n_launch = launches_per_step * args.steps
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    phases = {n: (v[0] * args.steps, v[1] * args.steps) for n, v in phases.items()}
    # the job is as slow as its slowest rank; requests mode: each rank serves its own
    # request (weak scaling); heads mode: all ranks serve one request (strong scaling)
    from paper_2602_02579_b200 import dist as pdist
    ms = pdist.max_over_ranks(ms, device="cuda")
    if world > 1:
        dist.barrier()
    value = (1 if shared else world) * s / (ms / 1e3)

    # ---- parity of this very run against the oracle fixture (rank 0's request)
    anchor = load_anchor(args, heads) if rank == 0 else None
    parity = anchor_parity(pipe, anchor, heads) if anchor is not None else None

    # ---- graph-timed phase split (each phase captured and replayed alone, serial)
    graph_phases = {}
    try:
        phase_fns = [("assemble_score_select", pipe.score_select), ("stage2", pipe.stage2)]
        if not pipe.fused_final:  # else the query rows ride along Stage II (pkv_recompute_query)
            phase_fns.append(("final", pipe.final))
        for name, fn in phase_fns:
            g = pipe.capture(fn)
            g.replay()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(args.steps):
                g.replay()
            a1.record(stream)
            torch.cuda.synchronize()
            graph_phases[name] = round(a0.elapsed_time(a1) / args.steps, 3)
            del g
    except Exception as e:  # noqa: BLE001 -- informational split only
        graph_phases["error"] = f"{type(e).__name__}: {e}"

    # ---- roofline of every kernel group; the dominant one is reported
    hbm, tf_burst, tf_sust, peak_kind = _peaks()
    idx = pipe.idx[: pipe.k].cpu().numpy().astype(np.int64)
    k = pipe.k
    # per-rank work: this rank's heads / ffn slice when head-sharded
    if tokens:  # this rank's share of the selected rows (pkv_recompute_rows' unit assignment)
        from paper_2602_02579_b200 import tp as _tp
        idx = idx[_tp.rows_share(k, cfg.n_heads // cfg.n_kv_heads, world, rank)]
        k = int(idx.size)
    lcfg = dm.cache_config
    L, H, Hkv, dk, D = cfg.n_layers, lcfg.n_heads, lcfg.n_kv_heads, cfg.head_dim, cfg.hidden_dim
    F = cfg.ffn_dim // dm.tp_world
    lay = cfg.layout()
    work = {  # per launch group: (bound, algorithmic units, unit)
        "assemble": ("hbm", 4.0 * L * s * Hkv * lay.dkp * 2, "GB/s"),
        "qp_proj": ("hbm", dm.weight_bytes(include_head=False) / (4 * L), "GB/s"),
        "qp_attn": ("hbm", 2.0 * s * Hkv * dk * 2, "GB/s"),  # one layer's context K and V, 2 B each
        "rc_qkv": ("tensor", 2.0 * k * D * (H + 2 * Hkv) * dk, "TFLOP/s"),
        "rc_attn": ("tensor", 4.0 * H * dk * float(np.sum(idx + 1)), "TFLOP/s"),
        "rc_o": ("tensor", 2.0 * k * H * dk * D, "TFLOP/s"),
        "rc_gate_up": ("tensor", 2.0 * k * D * 2 * F, "TFLOP/s"),
        "rc_down": ("tensor", 2.0 * k * F * D, "TFLOP/s"),
        "lm_head": ("hbm", 2.0 * cfg.vocab_size * lay.Dp, "GB/s"),
    }
    rooflines = {}
    for name, (bound, units, unit) in work.items():
        tot_ms, cnt = phases[name]
        if cnt == 0 or tot_ms <= 0:
            continue
        if name == "lm_head":  # one GEMV per step, timed together with its final norm (2 timer scopes)
            cnt = args.steps
        if name == "qp_attn":  # one attention scope per layer per narrow pass (scoring [+ final])
            cnt = args.steps * L * (1 if pipe.fused_final else 2)
        per_launch_s = tot_ms / cnt / 1e3
        ach = units / per_launch_s / (1e9 if unit == "GB/s" else 1e12)
        peak = hbm if bound == "hbm" else tf_sust
        rooflines[name] = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                           "ms_per_launch": per_launch_s * 1e3, "launches": cnt}
    if "qp_attn" in rooflines:
        # the narrow attention implements fp32 math with fp16 plane products on the tensor
        # cores (s1_attn_tc.cu: 3 QK + 2 PV products, scoring pass 2 another 3 QK): its
        # executed tensor work against the bf16 peak, next to the algorithmic K/V bytes
        # above.  The scope holds both passes' kernels, combine and finish.
        r = rooflines["qp_attn"]
        R = args.m * (cfg.n_heads // cfg.n_kv_heads)
        prod = 2.0 * R * s * dk * Hkv * (5 + 3)  # pass 1 (3 QK + 2 PV) + pass 2 (3 QK)
        tf = prod / (r["ms_per_launch"] / 1e3) / 1e12
        r["executed_tensor"] = {"tflop_per_launch": prod / 1e12, "achieved": tf, "peak": tf_sust, "frac": tf / tf_sust,
                                "note": "latency-bound: one wave of 144 CTAs x 28 64-key tiles (DESIGN.md section 3)"}
    step_total = sum(v[0] for v in phases.values())
    dominant = max((n for n in rooflines), key=lambda n: phases[n][0])
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():  # ncu --set full capture of this workload's dominant kernel (per launch)
        traffic = json.loads(tfile.read_text()).get(args.config, {}).get(dominant) if not heads else None
    roof = dict(rooflines[dominant], kernel=dominant, traffic=traffic,
                peak_kind=f"{peak_kind} ({'sustained bf16' if rooflines[dominant]['bound'] == 'tensor' else 'HBM copy'})")
    floor = ttft_floor_ms(cfgd, args.p, args.m, hbm, tf_burst)

    line = {"metric": metric_name(cfgd, args.p), "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ttft_ms": ms, "higher_is_better": True,
            "scaling": "strong" if shared else "weak",
            "vs_baseline": None, "dtype": "fp16 (Stage II, fp32 accumulate) / fp32-faithful (narrow passes)",
            "data": ("synthetic: SYN1 random-init weights (reference init scale), token ids and chunk K/V, "
                     "reproduced bit for bit by the CPU oracle" if args.chunks == "synthetic" else
                     "synthetic: SYN1 random-init weights and token ids; chunk K/V precomputed on the GPU"),
            "config": arm_config(args, cfgd, world, heads, tokens),
            "gpu_launches": int(n_launch), "launch_mode": launch_mode,
            "clocks": clk, "roofline": roof,
            "ttft_floor_ms": round(floor, 2), "ttft_floor_frac": round(floor / ms, 4),
            "graph_phases_ms": graph_phases,
            "eager_phases_ms": {n: round(v[0], 3) for n, v in eager_phases.items()},
            "phases_ms": {n: round(v[0] / args.steps, 3) for n, v in phases.items()},
            "phase_share": {n: round(v[0] / step_total, 4) for n, v in phases.items() if step_total > 0},
            "kernel_rooflines": rooflines}
    if parity is not None:
        line["parity"] = parity
    if nccl_log is not None:
        line["nccl"] = nccl_summary(nccl_log)

    # ---- the north star's comparator: full GPU prefill of the same request, same kernels
    if args.full_steps > 0:
        pipe.full_prefill_step()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.full_steps):
            pipe.full_prefill_step()
        f1.record(stream)
        torch.cuda.synchronize()
        full_ms = pdist.max_over_ranks(f0.elapsed_time(f1) / args.full_steps, device="cuda")
        H, dk = cfg.n_heads, cfg.head_dim
        full_tf = 2.0 * s * dm.weight_bytes(include_head=False) * dm.tp_world / 2 + 4.0 * L * H * dk * s * (s + 1) / 2
        line["full_prefill"] = {"ttft_ms": full_ms, "tok_per_s": s / (full_ms / 1e3),
                                "ttft_ratio_full_over_prophet": full_ms / ms,
                                "tflops": full_tf / (full_ms / 1e3) / 1e12,
                                "what": "Stage II with all s context tokens selected (no chunk reuse) + finalize, "
                                        "eager launches"}

    # ---- BASELINE configs[3]: recompute-ratio sweep at the same context (graph-replayed)
    if args.p_sweep:
        sweep = {}
        for pp in [float(x) for x in args.p_sweep.split(",") if x.strip()]:
            if abs(pp - args.p) < 1e-12:
                sweep[f"{pp:g}"] = {"k": k, "ttft_ms": ms, "tok_per_s": s / (ms / 1e3)}
            else:
                sp_pipe = PrefillPipeline(dm, chunks, args.m, pp)
                sp_pipe.set_query(query)
                sp_pipe.step()
                try:
                    sp_pipe.capture()
                except Exception:  # noqa: BLE001 -- eager launches if the step cannot be captured
                    torch.cuda.synchronize()
                    sp_pipe.replay = sp_pipe.step
                sp_pipe.replay()
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                for _ in range(args.sweep_steps):
                    sp_pipe.replay()
                g1.record(stream)
                torch.cuda.synchronize()
                t_ms = pdist.max_over_ranks(g0.elapsed_time(g1) / args.sweep_steps, device="cuda")
                sweep[f"{pp:g}"] = {"k": sp_pipe.k, "ttft_ms": t_ms, "tok_per_s": s / (t_ms / 1e3),
                                    "ttft_floor_ms": round(ttft_floor_ms(cfgd, pp, args.m, hbm, tf_burst), 2)}
                del sp_pipe
                torch.cuda.empty_cache()
            if "full_prefill" in line:
                sweep[f"{pp:g}"]["ttft_ratio_full_over_prophet"] = line["full_prefill"]["ttft_ms"] / \
                    sweep[f"{pp:g}"]["ttft_ms"]
        line["p_sweep"] = sweep

    # ---- e2e through the public API with host (pinned) inputs
    if args.e2e_steps > 0:
        host = [(c._k_dev.cpu().pin_memory(), c._v_dev.cpu().pin_memory(), c.token_ids) for c in chunks]
        h2d = sum(a.numel() * 2 + b.numel() * 2 for a, b, _ in host)
        torch.cuda.synchronize()
        mw = dm

        def e2e_step():
            # host-tier chunk store: assemble() streams the pinned K/V to HBM layer by
            # layer, overlapped with the scoring pass
            dch = [P.ChunkKV.from_pinned(i, dm.fingerprint, ids, a, b, cfg.head_dim)
                   for i, (a, b, ids) in enumerate(host)]
            cache = P.assemble(dch, dm.cache_config, fp32_taps=False)
            sc = P.score_prophet(mw, cfg, cache, query)
            sel = P.select_top_p(sc, args.p)
            P.recompute_selected(mw, cfg, cache, P.RecomputePlan(sel))
            return P.finalize_query(mw, cfg, cache, query).first_logits

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ms = pdist.max_over_ranks((time.perf_counter() - t0) * 1e3 / args.e2e_steps, device="cuda")
        d2h = L * s * 4 + s * 4 + k * 4 + cfg.vocab_size * 4
        line["e2e"] = {"value": (1 if shared else world) * s / (e2e_ms / 1e3), "unit": "tok/s", "ms_per_step": e2e_ms,
                       "h2d_bytes_per_step": int(h2d + args.m * 8), "d2h_bytes_per_step": int(d2h),
                       "path": "assemble -> score_prophet -> select_top_p -> recompute_selected -> finalize_query, "
                               "chunk K/V copied from pinned host memory each step (layer-pipelined with "
                               "assembly and the scoring pass)"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ttft, tm, kk, n_s, wall = cpu_sample(cfgd, args.p, n_rows=args.ref_rows)
        line["cpu_baseline"] = {"value": s / ttft, "unit": "tok/s", "cores": cpu_cores(), "kind": "port",
                                "ttft_ms": ttft * 1e3, "threads": cpu_threads(),
                                "sample": f"oracle port of pikv: 1 layer, full width, s={s}, Stage II on {n_s}/{kk} "
                                          f"rows; extrapolated x{L} layers (sample wall {wall:.1f}s)",
                                "full_run": full_anchor_run(args)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
