timeout 300 python -m pytest tests/test_gpu_p2p_math.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for c in C4q C4s C4t; do python tools/profile_one.py $c 2 2>&1 | tail -1; done
