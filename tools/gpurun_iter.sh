# quick iteration on the GPU box: gpu tests, then the bench per workload
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for w in ${WORKLOADS:-headline cfg1 complement wr bernoulli}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload $w > gpurun_out/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$w.log
done
tail -3 gpurun_out/it_pytest.log
for w in ${WORKLOADS:-headline cfg1 complement wr bernoulli}; do python3 -c "
import json,sys
for l in open('gpurun_out/bench_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('%-12s %.3g samples/s  ms/step %.2f  kernel %.2f ms  split %.2f ms  frac %.3f  sm %s' % ('$w', d['value'], d['ms_per_step'], r['kernel_ms'], r['split_ms'], r['frac'], d['clocks']['sm_mhz']))
" ; tail -2 gpurun_out/bench_$w.log | grep -v "^{" ; done
