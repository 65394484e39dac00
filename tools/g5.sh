timeout 900 python tools/debug/lp_check.py > gpurun_out/g5_lp.txt 2>&1; echo "lp rc=$?"
cat gpurun_out/g5_lp.txt
