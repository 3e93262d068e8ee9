# source-level (SASS) stall samples of the two largest DFMA kernels
set -x
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_p2p_near_sym --launch-skip 2 -c 1 -f -o /tmp/srcn python tools/profile_step.py 4 > gpurun_out/srcpg.log 2>&1
ncu -i /tmp/srcn.ncu-rep --page source --csv > gpurun_out/srcpg_near5.csv 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_m2p_leaf2 --launch-skip 2 -c 1 -f -o /tmp/srcl python tools/profile_step.py 4 >> gpurun_out/srcpg.log 2>&1
ncu -i /tmp/srcl.ncu-rep --page source --csv > gpurun_out/srcpg_leaf5.csv 2>&1
ls -la gpurun_out/srcpg*
head -c 600 gpurun_out/srcpg_near5.csv
