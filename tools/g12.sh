timeout 900 python tools/debug/wide_check.py > gpurun_out/g12_wide.txt 2>&1; echo "rc=$?"
cat gpurun_out/g12_wide.txt
