cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "not full_size" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/it_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/it_bench.log
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/it_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_leaf" -c 1 -o gpurun_out/it_prof -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/it_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/it_ncu.log
