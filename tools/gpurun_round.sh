# Round measurement: gpu tests, smoke, default bench (full JSON), all workloads,
# launch list of the headline step, ncu --set full of each dominant kernel.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(nvidia-smi; nproc; lscpu | head -20) > gpurun_out/box.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/bench_reference.log
for w in cfg1 complement wr bernoulli bernoulli32 cfg0; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload $w > gpurun_out/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$w.log; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
for spec in "headline:k_leaf_warp_wor:3" "cfg1:k_leaf_warp_wor:3" "complement:k_leaf_bitmap_comp:1" "wr:k_leaf_warp_wr:3" "bernoulli:k_bernoulli:1"; do
  W=${spec%%:*}; rest=${spec#*:}; K=${rest%%:*}; S=${rest#*:}
  timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/plain_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/full_$W -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/ncu_full_$W.log 2>&1
done
tail -2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log
