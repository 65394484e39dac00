# Re-run the evidence pass's bench lines of every workload, the complement's
# ncu capture and the GPU parity subset for the bitmap path.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
rm -f gpurun_out/r2_bench_all.jsonl
for w in cfg0 cfg1 weak30 complement wr bernoulli bernoulli32 gnm algb; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w --cpu-seconds 6 >> gpurun_out/r2_bench_all.jsonl 2>> gpurun_out/r2_bench_all.err
done
for spec in complement:k_leaf_bitmap_comp; do
  W=${spec%%:*}; K=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o /tmp/r2_full_${W}_${K} -f \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/r2_ncu_${W}_${K}.log 2>&1
  R=/tmp/r2_full_${W}_${K}.ncu-rep
  ncu -i $R --page details --csv > gpurun_out/r2_full_${W}_${K}_details.csv 2>/dev/null
  ncu -i $R --page raw --csv > gpurun_out/r2_full_${W}_${K}_raw.csv 2>/dev/null
  ncu -i $R --page source --csv --print-source cuda,sass > gpurun_out/r2_full_${W}_${K}_source.csv 2>/dev/null
  gzip -f gpurun_out/r2_full_${W}_${K}_source.csv
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "complement or wor_full or gnm or bernoulli" > gpurun_out/r2_parity_subset.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r2_parity_subset.log
