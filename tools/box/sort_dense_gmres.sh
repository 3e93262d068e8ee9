# hand-written radix sort: binning/bucket tests, build time; ncu --set full of
# the dense kernel (N = 262,144) and of the GMRES kernels (config 2)
set -x
python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/sort_pytest.log 2>&1
tail -3 gpurun_out/sort_pytest.log
python tools/quick_time.py 4 > gpurun_out/sort_quick.log 2>&1
grep -E "build|apply" gpurun_out/sort_quick.log
python tools/dense_time.py > gpurun_out/dense_time.log 2>&1; cat gpurun_out/dense_time.log
ncu --set full --clock-control none --import-source on -k regex:k_direct -c 2 -o /tmp/dense_full python tools/dense_time.py > gpurun_out/dense_ncu.log 2>&1
ncu -i /tmp/dense_full.ncu-rep --page raw --csv > gpurun_out/r02_ncu_dense_raw.csv 2>&1
python tools/gmres_profile.py 60 > gpurun_out/gmres_time.log 2>&1; cat gpurun_out/gmres_time.log
ncu --set full --clock-control none --import-source on --launch-skip 400 -c 60 -o /tmp/gmres_full python tools/gmres_profile.py 60 > gpurun_out/gmres_ncu.log 2>&1
ncu -i /tmp/gmres_full.ncu-rep --page raw --csv > gpurun_out/r02_ncu_gmres_raw.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_build.csv -c 40 python tools/quick_time.py 4 > /dev/null 2>&1
ls -la gpurun_out | tail -12
