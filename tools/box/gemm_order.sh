set -x
python tools/quick_time.py 4 > gpurun_out/ord_quick.log 2>&1
tail -12 gpurun_out/ord_quick.log
python -m pytest tests/test_gpu_fullvec.py tests/test_gpu_parity.py -q -x > gpurun_out/ord_pytest.log 2>&1
tail -5 gpurun_out/ord_pytest.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_node_gemm -c 6 --csv --log-file gpurun_out/ord_gemm.csv python tools/quick_time.py 4 > gpurun_out/ord_ncu.log 2>&1
tail -30 gpurun_out/ord_gemm.csv
