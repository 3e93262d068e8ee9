set -x
for w in 2 4 8; do python tools/shard_time.py $w > gpurun_out/r02_shard_$w.txt 2>&1; done
python tools/cfg5_sweep.py > gpurun_out/r02_cfg5_sweep.csv 2> gpurun_out/r02_cfg5_sweep.err
python tools/stress_paths.py 11 24 > gpurun_out/r02_stress.txt 2>&1
STRESS_XGATE=1 python tools/stress_paths.py 5 16 > gpurun_out/r02_stress_xgate.txt 2>&1
tail -2 gpurun_out/r02_shard_*.txt
