# Round measurement, part a: gpu tests, smoke, default bench (full JSON), the
# reference arm, every workload, the launch list of the headline step.
# Part b (PART=b): ncu --set full of each dominant kernel, a few per call
# (tools/gpurun_round_full.sh; gpurun_out must stay under 64 MiB per call).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
[ "${PART:-a}" = "b" ] && exec bash tools/gpurun_round_full.sh
(nvidia-smi; nproc; lscpu | head -20) > gpurun_out/box.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/bench_reference.log
for w in cfg1 complement wr bernoulli bernoulli32 cfg0 gnm algb; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload $w > gpurun_out/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$w.log; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --launch-list > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --launch-list > gpurun_out/ncu_launch.log 2>&1
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log
