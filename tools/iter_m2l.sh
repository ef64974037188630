# M2L iteration: parity tests, then stage times of the default build and the variants
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/m2l_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/m2l_tests.log
CONFIGS="C4q C4s C4t C3 C5" bash tools/variants_gpu.sh 2>&1 | tee gpurun_out/m2l_variants.log
