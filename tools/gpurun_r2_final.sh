# Round-2 evidence pass (one gpurun call): GPU tests, bench lines of every
# workload, the headline launch list, ncu --set full of each dominant kernel,
# the paper-shaped sweep and the microbenchmarks.  Output: gpurun_out/r2_*.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem,power.limit --format=csv > gpurun_out/r2_box.txt 2>&1
nproc >> gpurun_out/r2_box.txt; lscpu | grep "Model name" >> gpurun_out/r2_box.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_box.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
python bench.py > gpurun_out/r2_bench_default.jsonl 2> gpurun_out/r2_bench_default.err
for w in cfg0 cfg1 weak30 complement wr bernoulli bernoulli32 gnm algb; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w --cpu-seconds 6 >> gpurun_out/r2_bench_all.jsonl 2>> gpurun_out/r2_bench_all.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.jsonl 2>&1
python bench.py --steps 2 --warmup 1 --launch-list --no-e2e --no-cpu > gpurun_out/r2_ll_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
      python bench.py --steps 2 --warmup 1 --launch-list --no-e2e --no-cpu > gpurun_out/r2_ll_ncu.log 2>&1
for spec in headline:k_leaf_warp_wor_sd_p2 cfg1:k_leaf_warp_wor_tu_p2 wr:k_leaf_warp_wr_p2 complement:k_leaf_bitmap_comp bernoulli:k_bernoulli headline:k_split_deep3 cfg1:k_split_coop cfg0:k_fused_wor_tu_p2 gnm:k_leaf_warp_gnm algb:k_bernoulli64d; do
  W=${spec%%:*}; K=${spec#*:}
  timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/r2_plain_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o /tmp/r2_full_${W}_${K} -f \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/r2_ncu_${W}_${K}.log 2>&1
  echo "$W $K ncu rc=$?" >> gpurun_out/r2_box.txt
  # export here (the reports are too large to bring back): details, raw, per-line source
  R=/tmp/r2_full_${W}_${K}.ncu-rep
  ncu -i $R --page details --csv > gpurun_out/r2_full_${W}_${K}_details.csv 2>/dev/null
  ncu -i $R --page raw --csv > gpurun_out/r2_full_${W}_${K}_raw.csv 2>/dev/null
  ncu -i $R --page source --csv --print-source cuda,sass > gpurun_out/r2_full_${W}_${K}_source.csv 2>/dev/null
  gzip -f gpurun_out/r2_full_${W}_${K}_source.csv
  if [ "$W" = headline ] && [ "$K" = k_leaf_warp_wor_sd_p2 ]; then cp $R gpurun_out/; fi
done
timeout 600 python tools/sweep.py > gpurun_out/r2_sweep.txt 2>&1
# the wide (u64-range) warp leaf at the sweep's n = 2^28 (N = 2^50)
python tools/debug/mid_calls.py 28 > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_warp_wide_wor -c 1 -o /tmp/r2_full_sweep28_k_leaf_warp_wide_wor -f \
      python tools/debug/mid_calls.py 28 > gpurun_out/r2_ncu_sweep28.log 2>&1
R=/tmp/r2_full_sweep28_k_leaf_warp_wide_wor.ncu-rep
ncu -i $R --page details --csv > gpurun_out/r2_full_sweep28_k_leaf_warp_wide_wor_details.csv 2>/dev/null
ncu -i $R --page raw --csv > gpurun_out/r2_full_sweep28_k_leaf_warp_wide_wor_raw.csv 2>/dev/null
ncu -i $R --page source --csv --print-source cuda,sass > gpurun_out/r2_full_sweep28_k_leaf_warp_wide_wor_source.csv 2>/dev/null
gzip -f gpurun_out/r2_full_sweep28_k_leaf_warp_wide_wor_source.csv
# memory-safety evidence (compute-sanitizer is closed on the pool): guard regions + checked build
[ -f build/var/librs_checked.so ] && bash tools/checked_suite.sh > gpurun_out/r2_checked.txt 2>&1
./tools/ubench/ubench > gpurun_out/r2_ubench.txt 2>&1
./tools/ubench/hgd_lat > gpurun_out/r2_hgd_lat.txt 2>&1
echo done >> gpurun_out/r2_box.txt
