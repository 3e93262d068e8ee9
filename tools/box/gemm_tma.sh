# node GEMM staged by TMA bulk copies: config-4 times, parity suites, ncu metrics of the kernel
set -x
python tools/quick_time.py 4 > gpurun_out/gtma_quick.log 2>&1
grep -E "apply|moments|far |near " gpurun_out/gtma_quick.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullvec.py -q -x > gpurun_out/gtma_pytest.log 2>&1
tail -3 gpurun_out/gtma_pytest.log
ncu --set full --clock-control none --import-source on -k regex:k_node_gemm -c 2 -f -o /tmp/gtma python tools/quick_time.py 4 > gpurun_out/gtma_ncu.log 2>&1
ncu -i /tmp/gtma.ncu-rep --page raw --csv > gpurun_out/r02_ncu_gemm_tma_raw.csv 2>&1
