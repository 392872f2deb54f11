timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/y_probe.py 6000 8
timeout 600 python tools/y_probe.py 20000 4
