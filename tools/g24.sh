timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_stats.py -x -q -k "bern or gnp or algb" > gpurun_out/g24_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g24_pytest.log
for w in bernoulli bernoulli32; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload $w > gpurun_out/g24_$w.json 2>&1; python3 -c "
import json
for l in open('gpurun_out/g24_$w.json'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$w', 'ms/step %.3f kernel %.3f frac %.3f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))
"; done
