for v in t0 t8; do
  IMQ_LIB_PATH=paper_2205_04194_b200/libimqfast_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_node_gemm --csv --log-file gpurun_out/c35_$v.csv python tools/shard_profile_rank.py 8 0 > /dev/null 2>&1
  echo $v; grep k_node_gemm gpurun_out/c35_$v.csv | tail -1 | awk -F'","' '{print $NF}'
  IMQ_LIB_PATH=paper_2205_04194_b200/libimqfast_$v.so python tools/shard_time.py 8 2>&1 | tail -1
done
