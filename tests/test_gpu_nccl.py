"""The NCCL back end of the head-sharded prefill, one process per GPU.

The two-rank cases run only where >= 2 GPUs are visible (this pool's boxes have one; the
in-process communicator in test_gpu_tp.py covers the sharded math there); the one-rank cases
drive the same NCCL calls (init, all-reduce, all-gather, graph capture) on one GPU.  `bench.py --gpus 2`
starts two ranks itself (torchrun), shards the KV heads over NCCL and checks its own
request against the CPU oracle fixture in-run; here the line must report two GPUs,
tensor parallelism, and a selection identical to the oracle's.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (NCCL over NVLink)")
def test_bench_two_ranks_nccl():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                          "--e2e-steps", "0", "--full-steps", "0", "--p-sweep", "", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=1800, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-4000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["config"]["parallelism"].startswith("tp2")
    assert line["scaling"] == "strong"
    if "parity" in line:
        assert line["parity"]["sel_ok"] and line["parity"]["pass"], line["parity"]


ALLREDUCE_SCRIPT = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["PKV_ROOT"])
import __graft_entry__; __graft_entry__.build()
from paper_2602_02579_b200 import tp
r = int(os.environ["RANK"]); torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
c = tp.nccl_comm()
W = dist.get_world_size()
for dt in (torch.float64, torch.float32, torch.bfloat16):
    x = torch.arange(100, dtype=dt, device="cuda") * (r + 1)
    c.allreduce_(x)
    torch.cuda.synchronize()
    assert torch.equal(x, torch.arange(100, dtype=dt, device="cuda") * (W * (W + 1) // 2)), dt
c.close()
dist.destroy_process_group()
print("ok", r)
'''

# token-parallel repair over an NCCL communicator (comm_allgather -> ncclAllGather), eager and
# replayed from a CUDA graph: every rank ends with the unsharded run's cache bit for bit
ROWS_SCRIPT = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["PKV_ROOT"]); sys.path.insert(0, os.path.join(os.environ["PKV_ROOT"], "tests"))
import __graft_entry__; __graft_entry__.build()
import paper_2602_02579_b200 as P
from paper_2602_02579_b200 import tp
from paper_2602_02579_b200.pipeline import PrefillPipeline
from test_gpu_parity import _materialise, _setup
r = int(os.environ["RANK"]); torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
cfg_o, seed, units, query, p = _materialise("c1")
w, chunks = _setup(cfg_o, seed, units, query)
cfg = P.ModelConfig(**cfg_o.json())
mw = P.ModelWeights(embed=w.embed, layers=[P.LayerWeights(**{n: getattr(lw, n) for n in (
    "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")}) for lw in w.layers],
    final_norm=w.final_norm, lm_head=w.lm_head)
dm = P.DeviceModel.from_host(mw, cfg)
dch = [P.ChunkKV(c.chunk_id, mw.fingerprint(cfg), c.token_ids, c.k_nr, c.v) for c in chunks]
one = PrefillPipeline(dm, dch, len(query), p); one.set_query(query); one.step()
c = tp.nccl_comm()
pipe = PrefillPipeline(dm.rows(c), dch, len(query), p); pipe.set_query(query)


def same():
    torch.cuda.synchronize()
    s = one.s
    for name in ("k_pool", "v_pool", "k2_pool"):
        assert torch.equal(getattr(pipe.cache, name)[:, :, :s], getattr(one.cache, name)[:, :, :s]), name
    assert torch.equal(pipe.logits, one.logits)


pipe.step(); same()
pipe.capture(); pipe.replay(); same()
del pipe
c.close()
dist.destroy_process_group()
print("ok", r)
'''


def _run_ranks(path, script, n, timeout=900):
    import os
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, PKV_ROOT=str(ROOT))
    path.write_text(script)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), str(path)],
                         capture_output=True, text=True, timeout=timeout, env=env)
    assert out.returncode == 0 and out.stdout.count("ok") == n, out.stderr[-4000:]


def test_nccl_allreduce_one_rank(tmp_path):
    """The NCCL binding on a one-GPU box: dlopen of torch's libnccl, the unique-id exchange,
    ncclCommInitRank and ncclAllReduce for every dtype the prefill uses (one-rank NCCL
    communicators are not short-circuited)."""
    _run_ranks(tmp_path / "nccl_rank.py", ALLREDUCE_SCRIPT, 1)


def test_nccl_allgather_one_rank(tmp_path):
    """ncclAllGather inside the token-parallel repair, eager and under CUDA-graph capture,
    on one GPU."""
    _run_ranks(tmp_path / "nccl_rows.py", ROWS_SCRIPT, 1)


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (NCCL over NVLink)")
def test_nccl_allreduce_two_processes(tmp_path):
    """pkv_comm over NCCL: f64, f32 and bf16 in-place sums across two processes."""
    _run_ranks(tmp_path / "nccl_rank.py", ALLREDUCE_SCRIPT, 2)


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (NCCL over NVLink)")
def test_bench_two_ranks_token_parallel():
    """`bench.py --gpus 2 --mode tokens`: replicated scoring, token-parallel Stage II over
    NCCL all-gathers; rank 0's request is checked against the oracle fixture in-run."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--mode", "tokens", "--steps", "2",
                          "--warmup", "1", "--e2e-steps", "0", "--full-steps", "0", "--p-sweep", "",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=1800, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-4000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["parallelism"].startswith("tokens2")
    if "parity" in line:
        assert line["parity"]["sel_ok"] and line["parity"]["pass"], line["parity"]


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (NCCL over NVLink)")
def test_nccl_allgather_two_processes(tmp_path):
    """The all-gather the token-parallel Stage II uses, driven through a two-rank
    token-parallel repair on tiny inputs: both ranks end with the unsharded run's cache bit
    for bit."""
    _run_ranks(tmp_path / "nccl_rows.py", ROWS_SCRIPT, 2)
