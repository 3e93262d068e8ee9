# node GEMM tile variants (development .so files built with IMQ_BUILD_TAG / IMQ_NVCC_EXTRA)
for v in ${VARIANTS:-g32_16_3 g64_16_2 g32_32_2 g64_16_3}; do
  echo "== $v"
  IMQ_LIB_PATH=paper_2205_04194_b200/libimqfast_$v.so python tools/quick_time.py 4 2>&1 | grep -E "^apply|^far "
  IMQ_LIB_PATH=paper_2205_04194_b200/libimqfast_$v.so ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_node_gemm -c 3 --csv --log-file gpurun_out/gv_$v.csv python tools/profile_step.py 4 > /dev/null 2>&1
  grep k_node_gemm gpurun_out/gv_$v.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(TreeParams.*)//'
done
