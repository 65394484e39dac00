./tools/ubench/ubench > gpurun_out/g4_ubench.txt 2>&1
python tools/debug/lp_prof.py > gpurun_out/g4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_leaf_lp -s 1 -c 1 -o gpurun_out/g4_lp python tools/debug/lp_prof.py > gpurun_out/g4_ncu.log 2>&1
echo "ncu rc=$?"
head -40 gpurun_out/g4_ubench.txt
