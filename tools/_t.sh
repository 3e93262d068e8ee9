timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
timeout 900 python tools/cheb_accuracy.py 2>&1 | tail -14
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
