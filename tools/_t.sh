timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
IMQ_FAR_NOLSPLIT=1 timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
timeout 300 python tools/quick_time.py 3 2>&1 | grep -E "apply"
IMQ_FAR_NOLSPLIT=1 timeout 300 python tools/quick_time.py 3 2>&1 | grep -E "apply"
timeout 900 python tools/cheb_accuracy.py 2>&1 | tail -13
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 2
