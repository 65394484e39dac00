# ncu --set full of each dominant kernel (a few per call: the reports are large)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for spec in ${SPECS:-headline:k_leaf_warp_wor:3 cfg1:k_leaf_warp_wor_tu:3 complement:k_leaf_bitmap_comp:1}; do
  W=${spec%%:*}; rest=${spec#*:}; K=${rest%%:*}; S=${rest#*:}
  timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/plain_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/full_$W -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/ncu_full_$W.log 2>&1
  echo "$W ncu rc=$?"
done
