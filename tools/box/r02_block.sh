# block product: tests, bench line, compute-sanitizer on a small block case
set -x
python -m pytest tests/test_gpu_parity.py -q -k "block or batch" > gpurun_out/blk_pytest.log 2>&1
tail -5 gpurun_out/blk_pytest.log
python bench.py > gpurun_out/blk_bench.json 2> gpurun_out/blk_bench.err
tail -c 600 gpurun_out/blk_bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/blk_bench.json'))
print(d['ms_per_step'], d['value'], d['e2e'], d['clocks'])
PY
