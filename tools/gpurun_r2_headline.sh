cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for spec in headline:k_leaf_warp_wor_sd_p2; do
  W=${spec%%:*}; K=${spec#*:}
  timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/r2_plain_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o /tmp/r2_full_${W}_${K} -f \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/r2_ncu_${W}_${K}.log 2>&1
  R=/tmp/r2_full_${W}_${K}.ncu-rep
  ncu -i $R --page details --csv > gpurun_out/r2_full_${W}_${K}_details.csv 2>/dev/null
  ncu -i $R --page raw --csv > gpurun_out/r2_full_${W}_${K}_raw.csv 2>/dev/null
  ncu -i $R --page source --csv --print-source cuda,sass > gpurun_out/r2_full_${W}_${K}_source.csv 2>/dev/null
  gzip -f gpurun_out/r2_full_${W}_${K}_source.csv
  cp $R gpurun_out/
done
python bench.py > gpurun_out/r2_bench_default.jsonl 2> gpurun_out/r2_bench_default.err
