#!/usr/bin/env python
"""Benchmark of the Sparse DNN inference loop on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C4] [--dtype f32|f64] [--scaling strong|weak]

A step is one pass of the whole network (all L layers plus the category
list) over the batch, the reference's timed region (engine.py:336-339).
Default workload: C4, the flagship (N=65536, L=1920, 60,000 rows), which
fits one B200.

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun environment
re-launches this script under `torch.distributed.run` with N ranks (NCCL on
GPUs, gloo without).  Every rank holds a full weight replica; by default
(`--scaling strong`, north_star) the one 60,000-row batch is split into
contiguous row blocks (the reference's data-parallel tiling,
engine.py:222,237-251) and `value` is the batch's edges over the slowest
rank's device time.  With N > 1 a `weak` field adds the other reading:
every rank a full batch of its own rows.  There is no per-layer
collective, only the final category gather and max-over-ranks reductions.

`value`: nominal edges/s (inputs x N x 32 x L / t, challenge.py:131-135)
with Y0 resident in HBM, device time from CUDA events on the engine's
stream.  `e2e`: the same metric through the C ABI with host buffers (the
reference's int64/float64 CSR in, H2D of Y0 and D2H of the categories
inside the timed region).  `roofline`: the dominant launch against
measured HBM bandwidth (`roofline.launches`: every launch of the step);
`live.pruned_columns`: (tile, output) columns proven empty from their line
bounds -- nothing is skipped unproven: every layer of every
live tile is still visited, results are bit-identical with pruning off.  `cpu_baseline` / `--impl reference`: the
UNMODIFIED reference engine (`sdnnbench.engine.infer_timed`, numba,
data-parallel over every host core, float64) from `baseline/_ref` on a
bounded sample of the same workload, extrapolated to the full batch (the
oracle's C port stands in only when the reference is not installed).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1909_05631_b200 import workloads as W  # noqa: E402
from paper_1909_05631_b200.dist import RankGroup, shard  # noqa: E402

METRIC = "edges/sec (inputs×N×32×L / time)"
UNIT = "edges/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
HBM_FALLBACK = 6650.0  # B200_PROFILING.md fallback, GB/s
REF_DIR = ROOT / "baseline" / "_ref"


def hbm_peak():
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK, "fallback"


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return "unknown"


# -------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.file = None

    def start(self):
        if self.device is None:
            return self
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

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


# ------------------------------------------------- CPU baseline (reference)

def reference_engine():
    """(sdnnbench.engine, sdnnbench.model) of the UNMODIFIED reference from
    baseline/_ref (offline pip install of /root/reference; travels to the
    GPU box with the repo), or None when it is not installed."""
    if not (REF_DIR / "sdnnbench" / "engine.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "sdnn_numba_cache"))
    if str(REF_DIR) not in sys.path:
        sys.path.append(str(REF_DIR))
    try:
        from sdnnbench import engine, model
    except Exception:  # noqa: BLE001 -- e.g. numba missing: the port stands in
        return None
    return engine, model


LEAD_LAYERS = 8    # layers timed on the row sample (as specified, rows die by layer 2-3)
DEAD_LAYERS = 16   # layers timed on the full batch of empty rows


def cpu_rows_for(w: W.Workload) -> int:
    if w.value > 0.1:  # live companions: rows saturate and stay dense
        return 64
    return {1024: 60000, 4096: 20000, 16384: 6000, 65536: 2000}.get(w.n, 2000)


class CpuBaseline:
    """The reference's inference loop on the host cores over a bounded
    sample of workload `w`, extrapolated to the full batch.

    A step times (a) the first `lead` layers over `S` rows of Y0 (rows are
    independent, engine.py:237-251), scaled by B/S, and (b) when every
    sampled row is dead after them, the remaining layers as `dead`
    distinct layers over the full B-row batch of empty rows (zero rows stay
    zero; their cost is the per-row loop of engine.py:81-83), scaled by
    (L - lead) / dead.  If sampled rows are still alive after the lead
    layers, (a) is scaled by L / lead instead.  `kind` "reference" runs
    sdnnbench.engine.infer_timed itself (mode data_parallel, one worker per
    host core, float64); "port" the oracle's C restatement (float64), used
    only when the reference is not installed."""

    def __init__(self, w: W.Workload, rows: int, threads: int, prefer: str = "reference"):
        self.w, self.threads = w, threads
        self.S = max(1, min(w.batch, rows))
        self.lead = min(w.layers, LEAD_LAYERS)
        self.dead = min(w.layers - self.lead, DEAD_LAYERS)
        layers = W.layers_csr(w, 0, self.lead + self.dead, threads)
        off, cols, vals = W.images(w, n_rows=self.S, threads=threads)
        ref = reference_engine() if prefer == "reference" else None
        self.kind = "reference" if ref else "port"
        if ref:
            self.RE, M = ref
            lw = [M.LayerWeights(M.SparseMatrix(w.n, w.n, *c, check=False), w.bias) for c in layers]
            self.lead_model = M.NetworkModel(w.n, tuple(lw[:self.lead]))
            self.dead_model = M.NetworkModel(w.n, tuple(lw[self.lead:])) if self.dead else None
            self.y0 = M.FeatureBatch(M.SparseMatrix(self.S, w.n, off, cols, vals, check=False))
            self.empty = M.FeatureBatch(M.SparseMatrix.empty(w.batch, w.n))
            self.cfg = self.RE.InferenceConfig(ymax=w.ymax, mode="data_parallel", workers=threads)
        else:
            from oracle import oracle as O

            self.O = O
            cs = [O.CSR(w.n, w.n, *c) for c in layers]
            self.lead_model, self.dead_model = cs[:self.lead], cs[self.lead:]
            self.y0 = O.CSR(self.S, w.n, off, cols, vals)
            self.empty = O.CSR(w.batch, w.n, np.zeros(w.batch + 1, np.int64), np.zeros(0, np.int64),
                               np.zeros(0))
        self.live_after = None

    def _timed(self, model, y):
        """(seconds, rows alive after) of one timed region: infer + categorize."""
        if self.kind == "reference":
            _, cats, sec = self.RE.infer_timed(model, y, self.cfg)
            return sec, len(cats)
        t0 = time.perf_counter()
        out = self.O.infer(model, [self.w.bias] * len(model), y, self.w.ymax, precision=64,
                           threads=self.threads)
        cats = self.O.categorize(out)
        return time.perf_counter() - t0, int(cats.size)

    def step(self) -> float:
        """Extrapolated seconds of one full-batch pass."""
        w = self.w
        t_lead, alive = self._timed(self.lead_model, self.y0)
        self.live_after = alive
        t = t_lead * w.batch / self.S
        if self.lead < w.layers:
            if alive == 0 and self.dead:
                t_dead, _ = self._timed(self.dead_model, self.empty)
                t += t_dead * (w.layers - self.lead) / self.dead
            else:
                t *= w.layers / self.lead
        return t

    def describe(self) -> str:
        w = self.w
        eng = ("sdnnbench.engine.infer_timed (the unmodified reference from baseline/_ref, numba), "
               f"mode=data_parallel, workers={self.threads}, float64"
               if self.kind == "reference" else
               f"oracle/ C port of engine.py:64-137,192-251 (reference not installed), {self.threads} "
               "threads, float64")
        s = f"{eng}; {self.S} of {w.batch} rows through layers 1-{self.lead}"
        if self.S < w.batch:
            s += f" x {w.batch / self.S:.1f} (rows)"
        if self.lead < w.layers:
            if self.live_after == 0 and self.dead:
                s += (f"; every sampled row dead after layer {self.lead}, so layers {self.lead + 1}-{w.layers}"
                      f" timed as {self.dead} layers over the full {w.batch}-row batch of empty rows"
                      f" x {(w.layers - self.lead) / self.dead:.1f} (layers)")
            else:
                s += f"; {self.live_after} sampled rows still alive, x {w.layers / self.lead:.1f} (layers)"
        extrap = self.S < w.batch or self.lead < w.layers
        return s + ("; extrapolated" if extrap else "; full workload") + f"; CPU: {cpu_model()}"


def cpu_baseline(w: W.Workload, rows: int = 0, prefer: str = "reference") -> dict:
    """One bounded CPU-baseline measurement for our line (rank 0, N=1):
    one untimed warm-up step (numba specialises on the read-only arrays)
    and one timed step."""
    threads = os.cpu_count() or 1
    cb = CpuBaseline(w, rows or cpu_rows_for(w), threads, prefer)
    cb.step()
    t = cb.step()
    return {"value": w.edges / t, "unit": UNIT, "cores": threads, "kind": cb.kind,
            "sample": cb.describe(), "seconds_extrapolated": t, "dtype": "f64"}


# ------------------------------------------------------------ our arm

class DeviceArm:
    """This rank's row block on its GPU through the product path
    (libsdnn.so via the package's DeviceNetwork).  Weights: with N > 1,
    rank 0 generates the device ELL and the others receive it by NCCL
    broadcast over NVLink/NVSwitch (untimed setup)."""

    def __init__(self, args, dist: RankGroup, w: W.Workload, r0: int, r1: int):
        import torch

        from paper_1909_05631_b200.engine import DeviceNetwork

        self.torch, self.args, self.dist, self.w = torch, args, dist, w
        self.device = dist.local
        self.rows = r1 - r0
        threads = host_threads()
        self.net = net = DeviceNetwork(w.n, self.device, args.dtype)
        weights = args.weights if args.weights != "auto" else ("broadcast" if dist.world > 1 else "generate")
        if w.kind == "radixnet":  # K1: RadiX-Net weights, digit-like images resized on the device
            net.add_radixnet_layers(w.weight_seed, 0, w.layers, w.value, w.bias)
            self.batch = net.upload_images(W.stroke_images(w.batch)[r0:r1], w.side)
            self.off, self.cols, self.vals = self.batch.to_csr()
            self.nnz0 = int(self.off[-1])
            return
        if weights == "broadcast" and dist.world > 1:
            if dist.rank == 0:
                net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias,
                                         threads=os.cpu_count() or 1)
            else:
                net.add_layers_uninit(w.layers, w.width, w.bias)
            dist.broadcast_layers(net, 0, w.layers)
        else:
            net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias, threads=threads)
        self.off, self.cols, self.vals = W.images(w, n_rows=self.rows, row0=r0, threads=threads)
        self.nnz0 = int(self.off[-1])
        self.batch = net.upload_csr(self.rows, self.off, self.cols, self.vals)

    def sync(self):
        self.torch.cuda.synchronize(self.device)

    def step(self):
        return self.net.run(self.batch, self.w.ymax)

    def extras(self, ms_per_step: float, steps: int) -> dict:
        """Roofline (per-launch CUDA events), e2e through the C ABI."""
        args, dist, w, net = self.args, self.dist, self.w, self.net
        elem = 8 if args.dtype == "f64" else 4
        net.set_layer_timing(True)
        prof = net.run(self.batch, w.ymax)
        net.set_layer_timing(False)
        lb = layer_bytes(w, elem, prof.live_rows, self.nnz0, self.rows)
        live_layers = np.nonzero(prof.live_rows[:-1] > 0)[0]
        peak, peak_kind = hbm_peak()
        live_ms = float(prof.layer_ms[live_layers].sum()) if live_layers.size else 0.0
        all_gbs = lb.sum() / (live_ms * 1e-3) / 1e9 if live_ms > 0 else 0.0
        # dominant launch of the timed steps: the bit-line first-layer launch
        # covers layer 1, the persistent launch the rest
        stage_ms = dist.max_array(self.stage_ms / steps)
        bin_first = stage_ms[1] > 0
        # the Y0 CSR read of layer 1's byte model happens in the densify launch
        # (bit-line tiles); the first-layer launch keeps the output write and
        # the weights
        rd0 = float(self.nnz0 * (4 + elem) + (self.rows + 1) * 8) if prof.live_rows[0] > 0 else 0.0
        launch_bytes = [rd0 if bin_first else 0.0, float(lb[0]) - rd0 if bin_first else 0.0,
                        float(lb[1:].sum() if bin_first else lb.sum())]
        names = ["densify_quad_kernel (Y0 -> bit-line tiles)" if bin_first else "densify_kernel (Y0 -> tiles)",
                 "bin_quad_kernel (layer 1, quad/oct bit-lines)",
                 f"net_kernel (layers {2 if bin_first else 1}-{w.layers}, persistent)"]
        dom = int(np.argmax(stage_ms))
        dom_gbs = launch_bytes[dom] / (stage_ms[dom] * 1e-3) / 1e9 if stage_ms[dom] > 0 else 0.0
        traffic = measured_traffic(w, self.rows, args.dtype, names[dom].split()[0])
        live_total = dist.sum(float(prof.live_rows[:-1].sum()))

        # end to end through the C ABI with host buffers (sdnn_infer_streamed,
        # the call engine.infer makes): host CSR conversion + H2D of Y0 in row
        # segments overlapped with the run of earlier segments, + D2H of the
        # category list
        e2e_ms = 0.0
        for i in range(steps + 1):
            t0 = time.perf_counter()
            r2 = net.infer_csr(self.rows, self.off, self.cols, self.vals, w.ymax, want_y=False)
            _ = r2.categories.copy()
            dt = (time.perf_counter() - t0) * 1e3
            if i > 0:  # first call grows the pinned staging buffer
                e2e_ms += dt
        e2e_ms = dist.max(e2e_ms / steps)
        t0 = time.perf_counter()
        b2 = net.upload_csr(self.rows, self.off, self.cols, self.vals)
        t1 = time.perf_counter()
        r3 = net.run(b2, w.ymax)
        _ = r3.categories.copy()
        t2 = time.perf_counter()
        b2.close()
        total_edges = self.total_edges
        return {
            "live": {
                "rows_entering_each_live_layer": [int(x) for x in prof.live_rows[:-1][live_layers][:8]],
                "live_layers": int(live_layers.size),
                "live_edges_per_s": live_total * w.n * w.width / (ms_per_step * 1e-3),
                # (tile, output) columns whose line bounds proved them all zero (no gather)
                "pruned_columns": int(prof.pruned),
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
                # every launch of the step against the same byte model
                "launches": [{"kernel": names[i].split()[0], "ms": round(float(stage_ms[i]), 3),
                              "algorithmic_bytes": launch_bytes[i],
                              "frac": (launch_bytes[i] / (stage_ms[i] * 1e-3) / 1e9 / peak) if stage_ms[i] > 0 else 0.0}
                             for i in range(3)],
                "launches_note": ("algorithmic bytes are the contract's dense byte model; a launch whose layers were "
                                  "proven empty from their line bounds (live.pruned_columns) gathers nothing, so its "
                                  "frac can exceed 1"),
                "all_live_layers_gbs": all_gbs,
                "live_layer_ms": [round(float(prof.layer_ms[l]), 3) for l in live_layers[:8]],
                "peak_kind": peak_kind,
            },
            "e2e": {
                "value": total_edges / (e2e_ms * 1e-3),
                "unit": UNIT,
                "h2d_bytes_per_step": int(r2.h2d_bytes),
                "d2h_bytes_per_step": (w.layers + 1) * 4 + int(r2.live_rows[-1]) * 4,
                "ms_per_step": e2e_ms,
                "segments": int(r2.segments),
                "unstreamed_upload_then_run_ms": [round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1)],
            },
        }

    def weak(self, steps: int) -> dict:
        """Weak-scaling reading (N > 1): every rank a full batch of its own
        distinct rows (rank g: rows g*B ... (g+1)*B - 1 of the seeded image
        stream), same network."""
        dist, w = self.dist, self.w
        off, cols, vals = W.images(w, n_rows=w.batch, row0=dist.rank * w.batch, threads=host_threads())
        b = self.net.upload_csr(w.batch, off, cols, vals)
        del off, cols, vals
        for _ in range(2):
            self.net.run(b, w.ymax)
        dist.barrier()
        self.sync()
        ms = sum(self.net.run(b, w.ymax).device_ms for _ in range(steps)) / steps
        self.sync()
        dist.barrier()
        b.close()
        ms = dist.max(ms)
        return {"value": w.edges * dist.world / (ms * 1e-3), "ms_per_step": ms,
                "global_batch": w.batch * dist.world, "steps": steps,
                "note": "every GPU a full batch of its own distinct rows"}

    def close(self):
        self.batch.close()
        self.net.close()


def run_ours(args, dist: RankGroup, arm_cls=None):
    """Generic rank logic: shard, warm up, time exactly K steps between
    barriers + device syncs, max over ranks, gather categories.  `arm_cls`
    is the per-rank executor (DeviceArm; the CPU tests inject a stand-in
    to exercise this logic under gloo)."""
    w = workload(args)
    if args.scaling == "weak":  # every rank a full batch of its own rows (rows are independent)
        r0, r1 = dist.rank * w.batch, (dist.rank + 1) * w.batch
    else:  # the batch row-partitioned over the ranks (engine._infer_data_parallel tiling)
        r0, r1 = shard(w.batch, dist.rank, dist.world)
    total_edges = w.edges * (dist.world if args.scaling == "weak" else 1)
    global_batch = w.batch * (dist.world if args.scaling == "weak" else 1)
    t_setup = time.perf_counter()
    arm = (arm_cls or DeviceArm)(args, dist, w, r0, r1)
    arm.total_edges = total_edges
    setup_s = time.perf_counter() - t_setup

    clocks = ClockSampler(getattr(arm, "device", None)).start()  # sampling by the timed region
    for _ in range(args.warmup):
        arm.step()
    dist.barrier()
    arm.sync()
    t_region0 = time.time()
    dev_ms, wall0, launches = 0.0, time.perf_counter(), 0
    stage_ms = np.zeros(3)
    for _ in range(args.steps):
        res = arm.step()
        dev_ms += res.device_ms
        launches += res.launches
        stage_ms += res.stage_ms
    arm.sync()
    wall_ms = (time.perf_counter() - wall0) * 1e3
    t_region1 = time.time()
    dist.barrier()
    clk = clocks.stop((t_region0, t_region1))
    arm.stage_ms = stage_ms
    ms_per_step = dist.max(dev_ms / args.steps)
    wall_per_step = dist.max(wall_ms / args.steps)
    cats = dist.gather_categories(res.categories, r0)

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
        "categories": int(cats.size),
        "gpu_launches": launches,
        "wall_ms_per_step": wall_per_step,
        "clocks": clk,
        "setup_s": dist.max(setup_s),
    }
    if hasattr(arm, "extras"):
        line.update(arm.extras(ms_per_step, args.steps))
    if dist.world > 1 and args.scaling == "strong" and hasattr(arm, "weak") and not args.no_weak:
        line["weak"] = arm.weak(min(args.steps, 5))
    if dist.world == 1 and hasattr(arm, "net"):
        if not args.no_images:
            images = images_e2e(args, w, arm.net)
            if images:
                line["e2e_images"] = images
    arm.close()
    if dist.world == 1 and arm_cls is None:
        if args.also_f64 and args.dtype == "f32":
            line["f64"] = f64_line(args, w)
        if args.companions:
            line["companions"] = companions(args)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu and w.kind == "permunion":
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_rows)
    return line


def f64_line(args, w: W.Workload) -> dict:
    """The same workload on the bit-exact float64 path (the reference's
    arithmetic), N=1: a second field beside the float32 headline."""
    from paper_1909_05631_b200.engine import DeviceNetwork

    net = DeviceNetwork(w.n, 0, "f64")
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    off, cols, vals = W.images(w)
    b = net.upload_csr(w.batch, off, cols, vals)
    for _ in range(3):
        net.run(b, w.ymax)
    steps = max(3, min(args.steps, 10))
    clocks = ClockSampler(0).start()
    t0 = time.time()
    runs = [net.run(b, w.ymax) for _ in range(steps)]
    clk = clocks.stop((t0, time.time()))
    ms = sum(r.device_ms for r in runs) / steps
    stage = sum(r.stage_ms for r in runs) / steps
    b.close()
    net.close()
    return {"value": w.edges / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "launch_ms": {"densify": round(float(stage[0]), 3), "bin_layer": round(float(stage[1]), 3),
                          "net": round(float(stage[2]), 3)},
            "categories": int(runs[-1].categories.size), "clocks": clk}


def images_e2e(args, w: W.Workload, net):
    """End to end from raw images: B seeded 28x28
    uint8 images (W.stroke_images) copied to the device, resized /
    thresholded / flattened there (sdnn_batch_from_images, the reference's
    ingest.resize_threshold_flatten) and run through the workload's network,
    categories back; beside it the same rows through the host-CSR call."""
    side = int(round(w.n ** 0.5))
    if side * side != w.n or side not in (32, 64, 128, 256):
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


def companions(args):
    """Live-row companions (default K2 at C5 depth: rows stay alive and
    saturate, so every layer carries the full batch): 2 warm-up steps, at
    least 3 timed steps with their own clock record."""
    from paper_1909_05631_b200.engine import DeviceNetwork

    out = []
    for spec in args.companions.split(","):
        name, _, L = spec.partition(":")
        w = W.CONFIGS[name]
        if L:
            w = w.with_(layers=int(L))
        net = DeviceNetwork(w.n, 0, args.dtype)
        t_setup = time.perf_counter()
        if w.kind == "radixnet":  # K1: RadiX-Net weights, digit-like images resized on the device
            net.add_radixnet_layers(w.weight_seed, 0, w.layers, w.value, w.bias)
            b = net.upload_images(W.stroke_images(w.batch), w.side)
            nnz0 = b.nnz()
        else:
            net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
            off, cols, vals = W.images(w)
            b = net.upload_csr(w.batch, off, cols, vals)
            nnz0 = int(off[-1])
        setup_s = time.perf_counter() - t_setup
        for _ in range(2):
            net.run(b, w.ymax)
        steps = 3
        clocks = ClockSampler(0).start()
        t0 = time.time()
        runs = [net.run(b, w.ymax) for _ in range(steps)]
        clk = clocks.stop((t0, time.time()))
        ms = sum(r.device_ms for r in runs) / steps
        r = runs[-1]
        net.set_compaction(0)  # the same run without live-row compaction, for comparison
        r0 = net.run(b, w.ymax)
        net.set_compaction(10)
        net.set_layer_timing(True)
        p = net.run(b, w.ymax)
        elem = 8 if args.dtype == "f64" else 4
        lb = layer_bytes(w, elem, p.live_rows, nnz0, w.batch)
        peak, _ = hbm_peak()
        mid = w.layers // 2
        gbs = lb[mid] / (p.layer_ms[mid] * 1e-3) / 1e9 if p.layer_ms[mid] > 0 else 0.0
        out.append({
            "workload": (f"{w.name}: N={w.n}, L={w.layers}, batch={w.batch}, w={w.value}, bias={w.bias}, "
                         + ("RadiX-Net preset seed 42 (radixnet.py:293-310), 28x28 digit-like images "
                            "resized to 256x256 on the device" if w.kind == "radixnet"
                            else f"perm-union weights, Bernoulli({w.p}) images")),
            "setup_s": setup_s,
            "value": w.edges / (ms * 1e-3),
            "ms_per_step": ms,
            "steps": steps,
            "clocks": clk,
            "live_rows_last_layer": int(p.live_rows[-2]),
            "categories": int(r.categories.size),
            "row_compactions": int(r.compactions),
            "pruned_columns": int(r.pruned),
            "ms_per_step_without_compaction": r0.device_ms,
            "steady_layer_ms": float(p.layer_ms[mid]),
            "steady_layer_gbs": gbs,
            "steady_layer_frac": gbs / peak,
        })
        b.close()
        net.close()
    return out


# ------------------------------------------------------ reference arm

def run_reference(args, dist: RankGroup):
    """The driver's reference arm: the reference's own CPU implementation of
    the path on the host cores (CpuBaseline), same workload/metric/unit.
    Under torchrun only rank 0 works and prints."""
    if dist.rank != 0:
        return None
    w = workload(args)
    threads = os.cpu_count() or 1
    cb = CpuBaseline(w, args.cpu_rows or cpu_rows_for(w), threads)
    for _ in range(max(1, args.warmup)):  # >= 1: numba specialises on the first real call
        cb.step()
    secs = [cb.step() for _ in range(args.steps)]
    t = sum(secs) / len(secs)
    value = w.edges / t
    return {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded perm-union weights, Bernoulli images; BASELINE.json config)",
        "config": {"workload": f"{w.name}: N={w.n}, L={w.layers}, batch={w.batch}, p={w.p}, "
                               f"w={w.value}, bias={w.bias}, ymax={w.ymax}",
                   "neurons": w.n, "layers": w.layers, "global_batch": w.batch,
                   "parallelism": f"host threads ({threads}); the reference has no GPU path"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": cb.kind,
                         "sample": cb.describe()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------- launch

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
    if args.weight_value is not None:
        kw["value"] = args.weight_value
    return w.with_(**kw) if kw else w


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int, argv) -> int:
    """Re-launch this script under torch.distributed.run with n ranks on
    this node (the driver's own launch line), return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *argv]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the init log shows every rank joining
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def parser():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--weights", choices=("auto", "generate", "broadcast"), default="auto",
                    help="N>1: rank 0 generates, NCCL broadcast to the others (auto), or every rank generates")
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong",
                    help="strong: one batch split over the GPUs (north_star); weak: every GPU a full batch")
    ap.add_argument("--no-weak", action="store_true", help="N>1: skip the extra weak-scaling field")
    ap.add_argument("--workload", default="C4", choices=sorted(W.CONFIGS))
    ap.add_argument("--dtype", choices=("f32", "f64"), default="f32")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--weight-value", type=float, default=None,
                    help="override the workload's weight value (0.125: the live K2 regime)")
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-images", action="store_true", help="skip the end-to-end-from-images line")
    ap.add_argument("--also-f64", dest="also_f64", action="store_true", default=None,
                    help="N=1, f32: add the workload on the float64 path (default for C4)")
    ap.add_argument("--no-f64", dest="also_f64", action="store_false")
    ap.add_argument("--companions", default="K2:120,K1",
                    help="comma list NAME[:LAYERS] of live companions ('' to skip)")
    return ap


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    args = parser().parse_args(argv)
    if args.also_f64 is None:
        args.also_f64 = args.workload == "C4" and not (args.layers or args.batch or args.p is not None
                                                       or args.weight_value is not None)
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if world == 0 and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus, argv))
    if world and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
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
