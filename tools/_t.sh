timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
IMQ_CHEB_EVAL_FMA=1 timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
timeout 900 python tools/cheb_accuracy.py 2>&1 | tail -13
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cheb_ring" -c 4 python tools/profile_step.py 2>&1 | grep -E "duration" | tail -n 2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 2
