"""Cost of materialising the final Y (sdnn_run_y + sdnn_result_y_csr) on a
live workload (K2 generator: rows saturate and stay alive)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1909_05631_b200 import workloads as W  # noqa: E402
from paper_1909_05631_b200.engine import DeviceNetwork  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 6000
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = W.CONFIGS["K2"].with_(layers=layers, batch=rows)
off, cols, vals = W.images(w)
net = DeviceNetwork(w.n, 0, "f32")
net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
b = net.upload_csr(rows, off, cols, vals)
for want in (False, True, False, True):
    t0 = time.perf_counter()
    r = net.run(b, w.ymax, want_y=want)
    t1 = time.perf_counter()
    nnz = int(r.y[0][-1]) if want else -1
    print(f"want_y={want} wall {1e3*(t1-t0):.1f} ms device {r.device_ms:.1f} ms nnz {nnz} cats {r.categories.size}")
