# A/B the variant builds in build/var on the sweep's wide sizes (tools/sweep.py)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for f in build/var/librs_*.so; do
  n=$(basename $f .so)
  RS_LIB=$PWD/$f timeout 300 python tools/sweep.py ${SWEEP_E:-24 26 28} 2>/dev/null | grep "^  2" | sed "s/^/$n /"
done
done
