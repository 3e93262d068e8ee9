set -x
python tools/cfg4_full_compare.py > gpurun_out/c10_cfg4_full.json 2> gpurun_out/c10_cfg4_full.err
python tools/ref_sample_time.py 16777216 8 4096 4096 16 3 > gpurun_out/c10_ref_sample.json 2>&1
python tools/ref_sample_time.py 262144 5 1024 1024 16 3 > gpurun_out/c10_ref_sample_small.json 2>&1
python tools/gmres_protocol.py --ref > gpurun_out/c10_gmres.json 2> gpurun_out/c10_gmres.err
lscpu > gpurun_out/c10_lscpu.txt
