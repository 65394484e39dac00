python tools/debug/bern_prof.py > gpurun_out/g10_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bernoulli -s 1 -c 1 -o gpurun_out/g10_bern python tools/debug/bern_prof.py > gpurun_out/g10_ncu.log 2>&1
echo "ncu rc=$?"
