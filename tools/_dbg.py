import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle import oracle as O
from paper_1909_05631_b200 import workloads as W
from paper_1909_05631_b200 import engine as E
def case(n, layers, rows, value, p=0.35):
    side = int(round(n ** 0.5))
    w = W.Workload("t", n, layers, rows, side, int(side * 0.625), p, -0.45, value=value)
    off, cols, vals = W.images(w)
    return w, O.CSR(rows, n, off, cols, vals), [O.CSR(n, n, *W.layer_csr(w, l)) for l in range(layers)]
for dtype in sys.argv[1:]:
    saved = dict(os.environ)
    w, y0, layers = case(4096, 5, 700, 0.12)
    net = E.DeviceNetwork(w.n, 0, dtype)
    net.add_permunion_layers(w.weight_seed, 0, w.layers, w.width, w.value, w.bias)
    batch = net.upload_csr(y0.n_rows, y0.off, y0.cols, y0.vals)
    r = net.run(batch, w.ymax, want_y=True)
    print(dtype, "live", r.live_rows, "nnz", r.y[0][-1])
    os.environ["SDNN_HOST_Y"] = "1"
    r = net.run(batch, w.ymax, want_y=True)
    print(dtype, "hosty live", r.live_rows, "nnz", r.y[0][-1])
    os.environ["SDNN_HOST_Y"] = "0"
    os.environ["SDNN_WAVE_ROWS"] = "300"
    r = net.run(batch, w.ymax, want_y=True)
    print(dtype, "waves live", r.live_rows, "nnz", r.y[0][-1])
    net.close()
    os.environ.clear(); os.environ.update(saved)
    print("env WAVE", os.environ.get("SDNN_WAVE_ROWS"))
