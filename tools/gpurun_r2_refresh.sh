# Final refresh: every workload's bench line, the default (headline) line with
# e2e / oracle baseline, and the ncu captures of the WOR leaf kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
rm -f gpurun_out/r2_bench_all.jsonl
python bench.py > gpurun_out/r2_bench_default.jsonl 2> gpurun_out/r2_bench_default.err
for w in cfg0 cfg1 weak30 complement wr bernoulli bernoulli32 gnm algb; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w --cpu-seconds 6 >> gpurun_out/r2_bench_all.jsonl 2>> gpurun_out/r2_bench_all.err
done
for spec in headline:k_leaf_warp_wor_sd_p2 cfg1:k_leaf_warp_wor_tu_p2; do
  W=${spec%%:*}; K=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o /tmp/r2_full_${W}_${K} -f \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/r2_ncu_${W}_${K}.log 2>&1
  R=/tmp/r2_full_${W}_${K}.ncu-rep
  ncu -i $R --page details --csv > gpurun_out/r2_full_${W}_${K}_details.csv 2>/dev/null
  ncu -i $R --page raw --csv > gpurun_out/r2_full_${W}_${K}_raw.csv 2>/dev/null
  ncu -i $R --page source --csv --print-source cuda,sass > gpurun_out/r2_full_${W}_${K}_source.csv 2>/dev/null
  gzip -f gpurun_out/r2_full_${W}_${K}_source.csv
done
python bench.py --steps 2 --warmup 1 --launch-list --no-e2e --no-cpu > gpurun_out/r2_ll_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
      python bench.py --steps 2 --warmup 1 --launch-list --no-e2e --no-cpu > gpurun_out/r2_ll_ncu.log 2>&1
timeout 600 python tools/sweep.py > gpurun_out/r2_sweep.txt 2>&1
echo done
