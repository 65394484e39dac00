for f in build/var/librs_*.so; do n=$(basename $f .so); echo "== $n"; RS_LIB=$PWD/$f timeout 300 python tools/sweep.py 2>&1 | tail -12; done > gpurun_out/g11_sweep.txt 2>&1
cat gpurun_out/g11_sweep.txt
