timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/g23_pytest.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/g23_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g23_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g23_smoke.log
for w in headline cfg0 cfg1 complement wr bernoulli; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload $w > gpurun_out/g23_$w.json 2>&1; python3 -c "
import json
for l in open('gpurun_out/g23_$w.json'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('%-10s ms/step %.3f  kernel %.3f  split %.3f  frac %.3f' % ('$w', d['ms_per_step'], r['kernel_ms'], r['split_ms'], r['frac'] or 0))
"; done
timeout 300 python tools/sweep.py > gpurun_out/g23_sweep.txt 2>&1; cat gpurun_out/g23_sweep.txt
