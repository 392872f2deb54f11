"""The N>1 path on CPU: world_size-2 gloo process group running bench.py's
own rank logic (bench.run_ours: row shards, warm-up, timed steps between
barriers, max over ranks, category gather).  The per-rank executor injected
here computes with the CPU oracle (test infrastructure standing in for the
GPU); the product kernels are exercised by the GPU tests."""

import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest
import torch.multiprocessing as mp

import bench
from paper_1909_05631_b200 import workloads as W
from paper_1909_05631_b200.dist import RankGroup, shard

ROOT = Path(__file__).resolve().parent.parent
ARGS = ["--workload", "C1", "--layers", "4", "--batch", "203", "--weight-value", "0.125",
        "--steps", "2", "--warmup", "1", "--no-cpu", "--companions", ""]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleArm:
    """bench.DeviceArm's interface, computed by the oracle on the host."""

    device = None

    def __init__(self, args, dist, w, r0, r1):
        from oracle import oracle as O
        self.O, self.w, self.r0 = O, w, r0
        off, cols, vals = W.images(w, n_rows=r1 - r0, row0=r0)
        self.y0 = O.CSR(r1 - r0, w.n, off, cols, vals)
        self.layers = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
        self.rank = dist.rank

    def sync(self):
        pass

    def step(self):
        t0 = time.perf_counter()
        out = self.O.infer(self.layers, [self.w.bias] * self.w.layers, self.y0, self.w.ymax)
        ms = (time.perf_counter() - t0) * 1e3 + 1000.0 * (self.rank + 1)  # rank 1 is the slowest
        return SimpleNamespace(categories=self.O.categorize(out), device_ms=ms, launches=1,
                               stage_ms=np.array([0.0, 0.0, ms]))

    def close(self):
        pass


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    g = RankGroup(backend="gloo")
    line = bench.run_ours(bench.parser().parse_args(ARGS), g, arm_cls=OracleArm)
    stages = g.max_array(np.array([rank, 10.0 - rank, 3.0]))
    g.barrier()
    if rank == 0:
        q.put((line, stages.tolist()))
    g.close()


def test_shard_covers_rows_once():
    for batch in (0, 1, 7, 60000, 240000):
        for world in (1, 2, 3, 8):
            spans = [shard(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1


@pytest.mark.timeout(300)
def test_two_rank_gloo_bench_rank_logic_matches_single_process():
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    line, stages = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = bench.workload(bench.parser().parse_args(ARGS))
    off, cols, vals = W.images(w)
    layers = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
    want = O.categorize(O.infer(layers, [w.bias] * w.layers, O.CSR(w.batch, w.n, off, cols, vals)))
    assert want.size > 0
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["categories"] == want.size
    assert line["config"]["global_batch"] == w.batch
    assert line["ms_per_step"] >= 2000.0  # the slowest rank's time
    assert line["value"] == pytest.approx(w.edges / (line["ms_per_step"] * 1e-3))
    assert line["gpu_launches"] == 2
    assert stages == [1.0, 10.0, 3.0]  # per-launch times: elementwise max over ranks


@pytest.mark.timeout(600)
def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` (no torchrun env) re-launches itself with
    two ranks (gloo here); the reference arm prints from rank 0 with n_gpus 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--workload", "C1", "--batch", "2000", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=580, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_bench_refuses_mismatched_world():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--steps", "1"],
                         capture_output=True, text=True, timeout=120, cwd=str(ROOT), env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
