# A/B the variant builds in build/var: headline / cfg1 step time (median of 20)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for f in build/var/librs_*.so; do
  n=$(basename $f .so)
  for w in ${WORKLOADS:-headline cfg1}; do
    RS_LIB=$PWD/$f timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --workload $w 2>/dev/null | tail -1 | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('%-14s %-10s median %.3f  mean %.3f  leaf %.3f' % ('$n','$w', d['step_ms']['median'], d['ms_per_step'], r['kernel_ms']))"
  done
done
done
