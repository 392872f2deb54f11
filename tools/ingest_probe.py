"""Time the device weight ingest (CSR -> ELL) per C4 layer, warm."""
import sys
import time

sys.path.insert(0, ".")
from paper_1909_05631_b200 import workloads as W  # noqa: E402
from paper_1909_05631_b200.engine import DeviceNetwork  # noqa: E402
from paper_1909_05631_b200.model import SparseMatrix  # noqa: E402

w = W.CONFIGS["C4"]
net = DeviceNetwork(w.n, 0, "f32")
lay = [SparseMatrix(w.n, w.n, *W.layer_csr(w, l), check=False) for l in range(6)]
for i, m in enumerate(lay):
    t0 = time.perf_counter()
    net.add_layer_csr(m, w.bias)
    print(f"layer {i}: {1e3 * (time.perf_counter() - t0):.2f} ms")
