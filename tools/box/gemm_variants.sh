for v in g32_8_2 g16_16_2 g64_16_2 g32_8_3 g32_16_2; do
  IMQ_LIB_PATH=paper_2205_04194_b200/libimqfast_$v.so ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_node_gemm --csv --log-file gpurun_out/c24_$v.csv python tools/profile_step.py 4 > /dev/null 2>&1
  echo $v; grep k_node_gemm gpurun_out/c24_$v.csv | tail -2 | awk -F'","' '{print $(NF-2), $NF}'
done
