timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
IMQ_FAR_NOINNER=1 timeout 300 python tools/quick_time.py 4 2>&1 | grep -E "apply"
timeout 900 python tools/cheb_accuracy.py 2>&1 | tail -13
for sd in 7 11 13 17 23; do STRESS_COMPARE=1 timeout 900 python tools/stress_paths.py $sd 40; done > gpurun_out/stress_i14.txt 2>&1
for sd in 31 37; do STRESS_XGATE=1 STRESS_COMPARE=1 timeout 900 python tools/stress_paths.py $sd 30; done > gpurun_out/xgate_i14.txt 2>&1
echo "stress max $(grep -h ' dev ' gpurun_out/stress_i14.txt | awk '{for(i=1;i<=NF;i++) if($i=="dev") print $(i+1)}' | sort -g | tail -1)  xgate max $(grep -h ' dev ' gpurun_out/xgate_i14.txt | awk '{for(i=1;i<=NF;i++) if($i=="dev") print $(i+1)}' | sort -g | tail -1)"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 1
