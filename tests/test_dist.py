"""The N>1 path on CPU: world_size-2 gloo process group, rows sharded the
way bench.py shards them, categories gathered, time max-reduced.  The
per-rank compute stand-in is the CPU oracle (test infrastructure); the
product kernels are exercised by the GPU tests."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1909_05631_b200 import workloads as W
from paper_1909_05631_b200.dist import RankGroup, shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from oracle import oracle as O
    g = RankGroup(backend="gloo")
    w = W.CONFIGS["C1"].with_(layers=4, batch=203, value=0.125)
    r0, r1 = shard(w.batch, g.rank, g.world)
    off, cols, vals = W.images(w, n_rows=r1 - r0, row0=r0)
    layers = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
    out = O.infer(layers, [w.bias] * w.layers, O.CSR(r1 - r0, w.n, off, cols, vals), w.ymax)
    cats = g.gather_categories(O.categorize(out), r0)
    slowest = g.max(float(rank + 1))
    total = g.sum(float(r1 - r0))
    stages = g.max_array(np.array([rank, 10.0 - rank, 3.0]))
    g.barrier()
    if rank == 0:
        q.put((cats.tolist(), slowest, total, stages.tolist()))
    g.close()


def test_shard_covers_rows_once():
    for batch in (0, 1, 7, 60000, 240000):
        for world in (1, 2, 3, 8):
            spans = [shard(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_single_process():
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    cats, slowest, total, stages = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.CONFIGS["C1"].with_(layers=4, batch=203, value=0.125)
    off, cols, vals = W.images(w)
    layers = [O.CSR(w.n, w.n, *W.layer_csr(w, l)) for l in range(w.layers)]
    want = O.categorize(O.infer(layers, [w.bias] * w.layers, O.CSR(w.batch, w.n, off, cols, vals)))
    assert cats == want.tolist() and len(cats) > 0
    assert slowest == 2.0 and total == w.batch
    assert stages == [1.0, 10.0, 3.0]  # per-launch times: elementwise max over ranks
