# A/B the variant builds in build/var on one workload (kernel ms from bench)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in build/var/librs_*.so; do
  n=$(basename $f .so)
  for w in ${WORKLOADS:-headline}; do
    RS_LIB=$PWD/$f timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e ${CHECK:-} --workload $w > gpurun_out/var_${n}_$w.log 2>&1
    python3 -c "
import json
for l in open('gpurun_out/var_${n}_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('%-14s %-10s ms/step %.2f  leaf %.2f  frac %.3f' % ('$n','$w', d['ms_per_step'], r['kernel_ms'], r['frac']))
" || tail -2 gpurun_out/var_${n}_$w.log
  done
done
