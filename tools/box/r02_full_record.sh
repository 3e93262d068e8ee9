# Round-2 record: full GPU suite, bench (both arms), launch list, ncu summaries
# (the .ncu-rep files are reduced to CSV on the box: gpurun returns <= 64 MB)
set -x
python -m pytest tests -m gpu -q > gpurun_out/r02_pytest.log 2>&1
tail -3 gpurun_out/r02_pytest.log
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python tools/profile_step.py 4 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/r02_far_metrics.csv python tools/profile_step.py 4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -f -o /tmp/r02_full python tools/profile_step.py 4 > gpurun_out/r02_ncu_full.log 2>&1
ncu -i /tmp/r02_full.ncu-rep --page details --csv > gpurun_out/r02_ncu_full_details.csv 2>&1
ncu -i /tmp/r02_full.ncu-rep --page raw --csv > gpurun_out/r02_ncu_full_raw.csv 2>&1
python tools/shard_time.py 2 > gpurun_out/r02_shard_2.txt 2>&1
python tools/shard_time.py 4 > gpurun_out/r02_shard_4.txt 2>&1
python tools/shard_time.py 8 > gpurun_out/r02_shard_8.txt 2>&1
tail -1 gpurun_out/r02_shard_2.txt gpurun_out/r02_shard_4.txt gpurun_out/r02_shard_8.txt
ls -la gpurun_out
du -sh gpurun_out
