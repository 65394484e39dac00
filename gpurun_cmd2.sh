cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -v -rf --timeout 300 --durations=0 -k "not full_size" > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 900 python -m pytest tests -m gpu -v -rf --timeout 400 --durations=0 -k "full_size" > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leaf|k_split" -c 3 -o gpurun_out/prof1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu1.log
tail -5 gpurun_out/pytest_gpu2.log gpurun_out/pytest_gpu3.log gpurun_out/ncu1.log
