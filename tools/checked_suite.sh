# Memory-safety evidence without compute-sanitizer (closed on the pool):
# the GPU parity + guard-region suites against the normal build, then again
# against a build with the shared-memory index checks on (-DRS_CHECKED: a
# violation sets bit 8 of the device error word, which the tests assert is 0).
# Build the variant first: python tools/variants.py checked:RS_CHECKED
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_guards.py -q > gpurun_out/guards.log 2>&1; echo "guards rc=$?"; tail -2 gpurun_out/guards.log
RS_LIB=$PWD/build/var/librs_checked.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q > gpurun_out/checked.log 2>&1
echo "checked rc=$?"; tail -2 gpurun_out/checked.log
