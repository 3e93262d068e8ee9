for v in s0 s1024 s4096 s16384; do
  IMQ_LIB_PATH=paper_2205_04194_b200/libimqfast_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_m2m_tr" --csv --log-file gpurun_out/c32_$v.csv python tools/profile_step.py 4 > /dev/null 2>&1
  echo $v $(python tools/launch_summary.py gpurun_out/c32_$v.csv 2>/dev/null | head -3 | tr '\n' ' ')
  IMQ_LIB_PATH=paper_2205_04194_b200/libimqfast_$v.so python bench.py --no-gmres --no-cpu --steps 10 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  step', d['ms_per_step'], 'moments', d['roofline']['moments_ms'])"
done
