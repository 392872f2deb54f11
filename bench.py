#!/usr/bin/env python
"""Benchmark of the Sparse DNN inference loop on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C4] [--dtype f32|f64]

A step is one pass of the whole network (all L layers plus the category
list) over the batch, the reference's timed region (engine.py:336-339).
Default workload: C4, the flagship (N=65536, L=1920, 60,000 rows), which
fits one B200.  With N GPUs (torchrun, one process per GPU) every rank holds
a full weight replica; rows are independent, so by default (--scaling weak)
every rank runs a full batch of its own distinct rows and `value` counts the
rows of all ranks; --scaling strong splits one batch into contiguous row
blocks (the reference's data-parallel tiling).  There is no per-layer
collective, only the final category gather and a max-over-ranks of the
device time.

`value`: nominal edges/s (inputs x N x 32 x L / t, challenge.py:131-135) with
Y0 already resident in HBM, device time from CUDA events on the engine's
stream.  `e2e`: the same metric through the C ABI with host buffers (H2D of
Y0 and D2H of the categories inside the timed region).  `e2e_images`: the
same network fed raw 28x28 images resized on the device (the reference's
ingest.resize_threshold_flatten).  `roofline`: the
dominant layer launch against measured HBM bandwidth.  `cpu_baseline`: the
oracle port (a C restatement of the reference engine, oracle/) on the host
cores over a row sample.  `--impl reference` prints that CPU arm alone.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1909_05631_b200 import workloads as W  # noqa: E402

METRIC = "edges/sec (inputs×N×32×L / time)"
UNIT = "edges/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
HBM_FALLBACK = 6650.0  # B200_PROFILING.md fallback, GB/s


def hbm_peak():
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK, "fallback"


# -------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self, window=None):
        """Summarise the samples; with window=(t0, t1) (time.time() of the
        timed region) only samples inside it count, unless none fell inside
        (a very short region), then every sample taken under load counts."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.file.flush()
        rows = [ln.split(",") for ln in Path(self.file.name).read_text().splitlines() if ln.strip()]
        os.unlink(self.file.name)
        scope = "all"
        if window is not None:
            import datetime

            def ts(r):
                try:
                    return datetime.datetime.strptime(r[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except Exception:  # noqa: BLE001
                    return None
            inside = [r for r in rows if ts(r) is not None and window[0] <= ts(r) <= window[1]]
            if inside:
                rows, scope = inside, "timed region"
            else:
                scope = "warm-up + timed region (timed region shorter than the sampling period)"
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for name, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows), "scope": scope}


# ---------------------------------------------------------- distributed

from paper_1909_05631_b200.dist import RankGroup, shard  # noqa: E402


# ----------------------------------------------------------- byte model

def layer_bytes(w: W.Workload, elem: int, live: np.ndarray, nnz0: int, rows: int) -> np.ndarray:
    """Algorithmic HBM bytes of each layer launch (byte model):
    layer 1 reads Y0 as CSR (int32 column + value per entry, int64 offsets),
    later layers read the live dense rows; every live layer writes its dense
    output rows and reads the layer's ELL weights once (int32 + value per
    slot).  A layer with no live rows moves nothing."""
    out = np.zeros(w.layers)
    for l in range(w.layers):
        R = int(live[l])
        if R == 0:
            continue
        rd = nnz0 * (4 + elem) + (rows + 1) * 8 if l == 0 else elem * w.n * R
        out[l] = rd + elem * w.n * R + (4 + elem) * w.width * w.n
    return out


def measured_traffic(w: W.Workload, rows: int, dtype: str, kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture of this exact workload (profiles/traffic.json, written by
    tools/traffic_json.py), or None when no capture matches."""
    try:
        d = json.loads((ROOT / "profiles" / "traffic.json").read_text())
    except Exception:  # noqa: BLE001
        return None
    for e in d.get("captures", []):
        if (e.get("kernel") == kernel and e.get("n") == w.n and e.get("rows") == rows
                and e.get("dtype") == dtype and e.get("workload") == w.name and e.get("layers") == w.layers):
            return {"bytes": float(e["dram_bytes"]), "source": e["source"]}
    return None


# ------------------------------------------------------------ CPU oracle

def cpu_sample(w: W.Workload, rows: int, precision: int, threads: int):
    """Time the oracle port (C restatement of the reference engine) on a
    `rows`-row sample through all L layers; weights are generated per layer
    batch outside the clock (the reference loads its model before timing)."""
    from oracle import oracle as O
    from paper_1909_05631_b200 import _lib

    off, cols, vals = W.images(w, n_rows=rows)
    y = O.CSR(rows, w.n, off, cols, vals)
    g = _lib.gen()
    t_compute = 0.0
    batch = max(1, threads)
    idx = np.zeros((batch, w.n, w.width), np.int32)
    ones = np.full(w.n * w.width, w.value, np.float64)

    def to_csr(i):
        o = np.zeros(w.n + 1, np.int64)
        c = np.zeros(w.n * w.width, np.int64)
        v = np.zeros(w.n * w.width, np.float64)
        _lib.check_gen(g.sdnn_gen_ell_to_csr(w.n, w.n, w.width, _lib.ptr(idx[i]), _lib.ptr(ones),
                                             _lib.ptr(o), _lib.ptr(c), _lib.ptr(v)))
        return O.CSR(w.n, w.n, o, c, v)

    with ThreadPoolExecutor(max_workers=batch) as pool:
        for l0 in range(0, w.layers, batch):
            m = min(batch, w.layers - l0)
            _lib.check_gen(g.sdnn_gen_permunion_ell_layers(w.weight_seed, l0, m, w.n, w.width,
                                                           threads, _lib.ptr(idx)))
            csrs = list(pool.map(to_csr, range(m)))
            for lw in csrs:
                t0 = time.perf_counter()
                y = O.infer([lw], [w.bias], y, w.ymax, precision=precision, threads=threads)
                t_compute += time.perf_counter() - t0
    return t_compute, O.categorize(y)


def cpu_rows_for(w: W.Workload) -> int:
    if w.value > 0.1:  # live companions: rows saturate and stay dense
        return 8
    return {1024: 20000, 4096: 4000, 16384: 1500, 65536: 400}.get(w.n, 400)


# ------------------------------------------------------------ our arm

def run_ours(args, dist: RankGroup):
    import torch

    from paper_1909_05631_b200.engine import DeviceNetwork

    w = workload(args)
    dev = dist.local
    if args.scaling == "weak":  # every rank a full batch of its own rows (rows are independent)
        r0, r1 = dist.rank * w.batch, (dist.rank + 1) * w.batch
    else:  # the batch row-partitioned over the ranks (engine._infer_data_parallel tiling)
        r0, r1 = shard(w.batch, dist.rank, dist.world)
    rows = r1 - r0
    total_edges = w.edges * (dist.world if args.scaling == "weak" else 1)
    global_batch = w.batch * (dist.world if args.scaling == "weak" else 1)
    elem = 8 if args.dtype == "f64" else 4
    threads = host_threads()
    t_setup = time.perf_counter()
    net = DeviceNetwork(w.n, dev, args.dtype)
    weights = args.weights if args.weights != "auto" else ("broadcast" if dist.world > 1 else "generate")
    if weights == "broadcast" and dist.world > 1:
        # rank 0 generates (with every host core), the others receive the
        # device ELL over NCCL (NVLink/NVSwitch): untimed setup, SURVEY.md 8e
        if dist.rank == 0:
            net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias,
                                     threads=os.cpu_count() or 1)
        else:
            net.add_layers_uninit(w.layers, w.width, w.bias)
        dist.broadcast_layers(net, 0, w.layers)
    else:
        net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias, threads=threads)
    off, cols, vals = W.images(w, n_rows=rows, row0=r0, threads=threads)
    nnz0 = int(off[-1])
    batch = net.upload_csr(rows, off, cols, vals)
    setup_s = time.perf_counter() - t_setup

    clocks = ClockSampler(dev)
    clocks.start()  # before the warm-up, so nvidia-smi is sampling by the timed region
    for _ in range(args.warmup):
        net.run(batch, w.ymax)
    dist.barrier()
    torch.cuda.synchronize(dev)
    t_region0 = time.time()
    dev_ms, wall0 = 0.0, time.perf_counter()
    launches = 0
    stage_ms = np.zeros(3)
    for _ in range(args.steps):
        res = net.run(batch, w.ymax)
        dev_ms += res.device_ms
        launches += res.launches
        stage_ms += res.stage_ms
    torch.cuda.synchronize(dev)
    wall_ms = (time.perf_counter() - wall0) * 1e3
    t_region1 = time.time()
    dist.barrier()
    clk = clocks.stop((t_region0, t_region1))
    ms_per_step = dist.max(dev_ms / args.steps)
    wall_per_step = dist.max(wall_ms / args.steps)
    cats = dist.gather_categories(res.categories, r0)
    live_total = dist.sum(float(res.live_rows[:-1].sum()))

    # profiling pass (untimed): per-layer events for the roofline
    net.set_layer_timing(True)
    prof = net.run(batch, w.ymax)
    net.set_layer_timing(False)
    lb = layer_bytes(w, elem, prof.live_rows, nnz0, rows)
    live_layers = np.nonzero(prof.live_rows[:-1] > 0)[0]
    peak, peak_kind = hbm_peak()
    live_ms = float(prof.layer_ms[live_layers].sum()) if live_layers.size else 0.0
    all_gbs = lb.sum() / (live_ms * 1e-3) / 1e9 if live_ms > 0 else 0.0
    # dominant launch of the timed steps (CUDA events on the engine's stream):
    # the bit-line first-layer launch covers layer 1, the persistent launch
    # the rest; its algorithmic bytes are those of the layers it ran
    stage_ms = dist.max_array(stage_ms / args.steps)
    bin_first = stage_ms[1] > 0
    launch_bytes = [0.0, float(lb[0]) if bin_first else 0.0, float(lb[1:].sum() if bin_first else lb.sum())]
    names = ["densify_kernel (Y0 -> tiles)", "bin_layer_kernel (layer 1, bit-line tiles)",
             f"net_kernel (layers {2 if bin_first else 1}-{w.layers}, persistent)"]
    dom = int(np.argmax(stage_ms))
    dom_gbs = launch_bytes[dom] / (stage_ms[dom] * 1e-3) / 1e9 if stage_ms[dom] > 0 else 0.0
    traffic = measured_traffic(w, rows, args.dtype, names[dom].split()[0])

    # end to end through the C ABI with host buffers (sdnn_infer_streamed,
    # the call engine.infer makes): host CSR conversion + H2D of Y0 in row
    # segments overlapped with the run of earlier segments, + D2H of the
    # category list
    e2e_ms = 0.0
    for i in range(args.steps + 1):
        t0 = time.perf_counter()
        r2 = net.infer_csr(rows, off, cols, vals, w.ymax, want_y=False)
        _ = r2.categories.copy()
        dt = (time.perf_counter() - t0) * 1e3
        if i > 0:  # first call grows the pinned staging buffer
            e2e_ms += dt
    e2e_ms = dist.max(e2e_ms / args.steps)
    h2d = r2.h2d_bytes
    d2h = (w.layers + 1) * 4 + int(r2.live_rows[-1]) * 4
    # the same call unstreamed, for the split: upload, then run
    t0 = time.perf_counter()
    b2 = net.upload_csr(rows, off, cols, vals)
    t1 = time.perf_counter()
    r3 = net.run(b2, w.ymax)
    _ = r3.categories.copy()
    t2 = time.perf_counter()
    b2.close()
    e2e_split = [round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1)]
    images = images_e2e(args, w, net) if dist.world == 1 else None

    line = {
        "metric": METRIC,
        "value": total_edges / (ms_per_step * 1e-3),
        "unit": UNIT,
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (seeded perm-union weights, Bernoulli images; BASELINE.json config)",
        "config": {
            "workload": f"{w.name}: N={w.n}, L={w.layers}, batch={w.batch}, p={w.p}, "
                        f"w={w.value}, bias={w.bias}, ymax={w.ymax}",
            "neurons": w.n, "layers": w.layers, "global_batch": global_batch,
            "parallelism": (f"dp{dist.world}: " + ("a full batch of distinct rows per GPU"
                            if args.scaling == "weak" else "contiguous row blocks of one batch")
                            + ", weight replica per GPU, no per-layer collective"),
            "l2": "inputs larger than L2 (Y0 CSR and weights exceed 126 MB; no flush)",
        },
        "live": {
            "rows_entering_each_live_layer": [int(x) for x in prof.live_rows[:-1][live_layers][:8]],
            "live_layers": int(live_layers.size),
            "live_edges_per_s": live_total * w.n * w.width / (ms_per_step * 1e-3),
            "categories": int(cats.size),
        },
        "roofline": {
            "bound": "hbm",
            "achieved": dom_gbs,
            "peak": peak,
            "unit": "GB/s",
            "frac": dom_gbs / peak,
            "traffic": traffic["bytes"] if traffic else None,
            "traffic_source": traffic["source"] if traffic else None,
            "kernel": names[dom],
            "per_launch_ms": float(stage_ms[dom]),
            "algorithmic_bytes": launch_bytes[dom],
            "launch_ms": {"densify": round(float(stage_ms[0]), 3), "bin_layer": round(float(stage_ms[1]), 3),
                          "net": round(float(stage_ms[2]), 3)},
            "all_live_layers_gbs": all_gbs,
            "live_layer_ms": [round(float(prof.layer_ms[l]), 3) for l in live_layers[:8]],
            "peak_kind": peak_kind,
        },
        "e2e": {
            "value": total_edges / (e2e_ms * 1e-3),
            "unit": UNIT,
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "ms_per_step": e2e_ms,
            "segments": int(r2.segments),
            "unstreamed_upload_then_run_ms": e2e_split,
        },
        "gpu_launches": launches,
        "wall_ms_per_step": wall_per_step,
        **({"e2e_images": images} if images else {}),
        "clocks": clk,
        "setup_s": setup_s,
    }
    batch.close()
    net.close()
    if args.companions and dist.world == 1:
        line["companions"] = companions(args, net_cls=DeviceNetwork)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        S = args.cpu_rows or cpu_rows_for(w)
        t_cpu, _ = cpu_sample(w, S, 64 if args.dtype == "f64" else 32, threads)
        line["cpu_baseline"] = {
            "value": S * w.n * w.width * w.layers / t_cpu,
            "unit": UNIT,
            "cores": threads,
            "kind": "port",
            "sample": f"{S} of {w.batch} rows through all {w.layers} layers, oracle/ C port of "
                      f"engine._spmm_kernel+_bias_relu_clamp_kernel, {threads} threads, "
                      f"{'float64' if args.dtype == 'f64' else 'float32'}",
            "seconds": t_cpu,
        }
    return line


def images_e2e(args, w: W.Workload, net):
    """End to end from raw images: B seeded 28x28
    uint8 images (W.stroke_images) copied to the device, resized /
    thresholded / flattened there (sdnn_batch_from_images, the reference's
    ingest.resize_threshold_flatten) and run through the workload's network,
    categories back; beside it the same rows through the host-CSR call."""
    side = int(round(w.n ** 0.5))
    if args.no_images or side * side != w.n or side not in (32, 64, 128, 256):
        return None
    pix = W.stroke_images(w.batch)
    b = net.upload_images(pix, side)  # warm-up; its CSR feeds the host-CSR comparison
    off, cols, vals = b.to_csr()
    b.close()
    ms = []
    for _ in range(max(1, min(args.steps, 5)) + 1):
        t0 = time.perf_counter()
        b = net.upload_images(pix, side)
        r = net.run(b, w.ymax)
        _ = r.categories.copy()
        ms.append((time.perf_counter() - t0) * 1e3)
        h2d = b.h2d_bytes
        b.close()
    t0 = time.perf_counter()
    r2 = net.infer_csr(w.batch, off, cols, vals, w.ymax, want_y=False)
    host_ms = (time.perf_counter() - t0) * 1e3
    assert np.array_equal(r.categories, r2.categories)
    e2e_ms = float(np.mean(ms[1:]))
    return {
        "workload": f"{w.batch} seeded 28x28 uint8 stroke images resized on the device to "
                    f"{side}x{side}, then {w.name}'s network",
        "value": w.edges / (e2e_ms * 1e-3),
        "unit": UNIT,
        "ms_per_step": e2e_ms,
        "h2d_bytes_per_step": int(h2d),
        "y0_nnz_per_row": float(off[-1]) / w.batch,
        "categories": int(r.categories.size),
        "same_rows_from_host_csr_ms": host_ms,
    }


def companions(args, net_cls):
    """Live-row companion (K2 at C5 depth): rows stay alive and saturate,
    so every layer carries the full batch.  One warm-up, one timed step."""
    out = []
    for spec in args.companions.split(","):
        name, _, L = spec.partition(":")
        w = W.CONFIGS[name]
        if L:
            w = w.with_(layers=int(L))
        net = net_cls(w.n, 0, args.dtype)
        net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
        off, cols, vals = W.images(w)
        b = net.upload_csr(w.batch, off, cols, vals)
        net.run(b, w.ymax)
        r = net.run(b, w.ymax)
        net.set_compaction(0)  # the same run without live-row compaction, for comparison
        r0 = net.run(b, w.ymax)
        net.set_compaction(10)
        net.set_layer_timing(True)
        p = net.run(b, w.ymax)
        elem = 8 if args.dtype == "f64" else 4
        lb = layer_bytes(w, elem, p.live_rows, int(off[-1]), w.batch)
        peak, _ = hbm_peak()
        mid = w.layers // 2
        out.append({
            "workload": f"{w.name}: N={w.n}, L={w.layers}, batch={w.batch}, w={w.value}",
            "value": w.edges / (r.device_ms * 1e-3),
            "ms_per_step": r.device_ms,
            "live_rows_last_layer": int(p.live_rows[-2]),
            "categories": int(r.categories.size),
            "row_compactions": int(r.compactions),
            "ms_per_step_without_compaction": r0.device_ms,
            "steady_layer_ms": float(p.layer_ms[mid]),
            "steady_layer_gbs": lb[mid] / (p.layer_ms[mid] * 1e-3) / 1e9 if p.layer_ms[mid] > 0 else 0,
            "steady_layer_frac": (lb[mid] / (p.layer_ms[mid] * 1e-3) / 1e9) / peak if p.layer_ms[mid] > 0 else 0,
        })
        b.close()
        net.close()
    return out


# ------------------------------------------------------ reference arm

def run_reference(args, dist: RankGroup):
    if dist.rank != 0:
        return None
    w = workload(args)
    threads = os.cpu_count() or 1
    S = args.cpu_rows or cpu_rows_for(w)
    prec = 64 if args.dtype == "f64" else 32
    for _ in range(args.warmup):
        cpu_sample(w, S, prec, threads)
    secs = [cpu_sample(w, S, prec, threads)[0] for _ in range(args.steps)]
    t = sum(secs) / len(secs)
    value = S * w.n * w.width * w.layers / t
    sample = (f"{S} of {w.batch} rows through all {w.layers} layers per step, oracle/ C port of "
              f"the reference engine (engine.py:64-137,192-251), {threads} threads")
    return {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (seeded perm-union weights, Bernoulli images; BASELINE.json config)",
        "config": {"workload": f"{w.name}: N={w.n}, L={w.layers}, batch={w.batch}, p={w.p}, "
                               f"w={w.value}, bias={w.bias}",
                   "neurons": w.n, "layers": w.layers, "global_batch": w.batch,
                   "parallelism": "host threads"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def host_threads() -> int:
    """Host threads per rank: the node's cores split over its local ranks."""
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    return max(1, (os.cpu_count() or 1) // local)


def workload(args) -> W.Workload:
    w = W.CONFIGS[args.workload]
    kw = {}
    if args.layers:
        kw["layers"] = args.layers
    if args.batch:
        kw["batch"] = args.batch
    if args.p is not None:
        kw["p"] = args.p
    return w.with_(**kw) if kw else w


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--weights", choices=("auto", "generate", "broadcast"), default="auto",
                    help="N>1: rank 0 generates, NCCL broadcast to the others (auto), or every rank generates")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: every GPU a full batch of its own rows; strong: one batch split over GPUs")
    ap.add_argument("--workload", default="C4", choices=sorted(W.CONFIGS))
    ap.add_argument("--dtype", choices=("f32", "f64"), default="f32")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-images", action="store_true", help="skip the end-to-end-from-images line")
    ap.add_argument("--companions", default="K2:120",
                    help="comma list NAME[:LAYERS] of live companions ('' to skip)")
    args = ap.parse_args(argv)
    os.environ.setdefault("OMP_NUM_THREADS", str(host_threads()))  # libsdnn's upload threads
    dist = RankGroup()
    try:
        line = run_reference(args, dist) if args.impl == "reference" else run_ours(args, dist)
        if line is not None and dist.rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
