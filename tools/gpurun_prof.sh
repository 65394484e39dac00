# ncu --set full of the leaf kernel of one bench workload (plain run first)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
W=${W:-headline}; K=${K:-k_leaf}; TAG=${TAG:-prof}
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-1} -c 1 -o gpurun_out/$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --workload $W > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
tail -2 gpurun_out/ncu_$TAG.log
