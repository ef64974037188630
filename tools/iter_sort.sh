# sort iteration: parity + full-size tree tests, then build times per config
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/sort_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sort_tests.log
for c in C4q C4s C4t C3 C5; do python tools/profile_one.py $c 3 2>&1 | tail -1; done | tee gpurun_out/sort_times.log
