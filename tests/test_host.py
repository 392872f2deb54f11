"""Host-side logic of the drop-in (CPU only)."""

import numpy as np
import pytest

import bench
from paper_1909_05631_b200 import engine as E
from paper_1909_05631_b200 import errors
from paper_1909_05631_b200.model import (
    CategorySet, FeatureBatch, LayerWeights, NetworkModel, SparseMatrix,
)


def test_config_validation_mirrors_reference():  # test_engine.py:239-256
    with pytest.raises(errors.ParameterError):
        E.InferenceConfig(ymax=0.0)
    with pytest.raises(errors.ParameterError):
        E.InferenceConfig(mode="warp")
    with pytest.raises(errors.ParameterError):
        E.InferenceConfig(workers=0)
    with pytest.raises(errors.ParameterError):
        E.InferenceConfig(pipeline_stages=0)
    with pytest.raises(errors.ParameterError):
        E.InferenceConfig(batch_tile=0)
    with pytest.raises(errors.ParameterError):
        E.InferenceConfig(dtype="bf16")
    cfg = E.InferenceConfig()
    assert (cfg.ymax, cfg.mode, cfg.workers, cfg.dtype) == (32.0, "serial", 1, "f64")


def test_error_codes_map_to_reference_classes():
    assert isinstance(errors.from_code(2, "x"), errors.ParameterError)
    assert isinstance(errors.from_code(3, "x"), errors.CapacityError)
    assert isinstance(errors.from_code(4, "x"), errors.ShapeError)


def test_stage_partition():  # engine.py:226-229
    assert E._stage_partition(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert E._stage_partition(5, 5) == [(i, i + 1) for i in range(5)]


def test_shape_errors_raised_before_any_device_work():
    w = SparseMatrix.from_dense(np.eye(4))
    model = NetworkModel(4, (LayerWeights(w, -0.1),))
    with pytest.raises(errors.ShapeError):
        E.infer(model, FeatureBatch(SparseMatrix.from_dense(np.ones((2, 5)))))
    with pytest.raises(errors.ParameterError):
        E.infer(model, FeatureBatch(SparseMatrix.from_dense(np.ones((2, 4)))),
                E.InferenceConfig(mode="pipeline", pipeline_stages=3))
    with pytest.raises(errors.ShapeError):
        E.spmm(FeatureBatch(SparseMatrix.from_dense(np.ones((1, 3)))), w)


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    w = SparseMatrix.from_dense(np.eye(4))
    model = NetworkModel(4, (LayerWeights(w, -0.1),))
    with pytest.raises(errors.CapacityError):
        E.infer(model, FeatureBatch(SparseMatrix.from_dense(np.ones((2, 4)))))


def test_result_types_follow_the_caller_family():
    sm, fb, cs = E._family(FeatureBatch(SparseMatrix.empty(1, 2)))
    assert (sm, fb, cs) == (SparseMatrix, FeatureBatch, CategorySet)


def test_bench_shards_and_byte_model():
    assert bench.shard(10, 0, 3) == (0, 4)
    assert bench.shard(10, 2, 3) == (8, 10)
    assert bench.shard(2, 3, 4) == (2, 2)
    from paper_1909_05631_b200 import workloads as W
    w = W.CONFIGS["C4"].with_(layers=4)
    live = np.array([100, 90, 0, 0, 0])
    b = bench.layer_bytes(w, 4, live, nnz0=1000, rows=100)
    assert b[2] == 0 and b[3] == 0
    assert b[1] == 4 * w.n * 90 * 2 + 8 * 32 * w.n
    assert b[0] == 1000 * 8 + 101 * 8 + 4 * w.n * 100 + 8 * 32 * w.n


def test_bench_reference_arm_line_on_cpu():
    """`bench.py --impl reference` (the driver's reference arm) runs on host
    cores only and prints the contract's JSON line: impl, cpu_baseline with
    its kind / cores / sample, an e2e object with zero copy bytes."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--workload", "C1",
                          "--batch", "3000", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=str(root))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "edges/s"
    assert line["higher_is_better"] is True and line["steps"] == 1 and line["warmup"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
