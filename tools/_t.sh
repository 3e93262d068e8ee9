timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_p2m_leaf_g" -c 2 python tools/profile_step.py 2>&1 | grep -E "duration" | tail -n 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 1
