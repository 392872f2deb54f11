"""Time the device image ingest (sdnn_batch_from_images) by stage size."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1909_05631_b200 import workloads as W  # noqa: E402
from paper_1909_05631_b200.engine import DeviceNetwork  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
pix = W.stroke_images(n)
for side in [int(s) for s in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["32", "256"])]:
    net = DeviceNetwork(side * side, 0, "f32")
    for i in range(4):
        t0 = time.perf_counter()
        b = net.upload_images(pix, side)
        t1 = time.perf_counter()
        b.close()
        if i:
            print(f"side {side}: upload_images {1e3 * (t1 - t0):.1f} ms")
    net.close()
