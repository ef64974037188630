# one GPU iteration after a kernel change: selected -m gpu tests, then per-config stage times
# usage: bash tools/gpu_iter.sh TAG "pytest selection" "C4q C4s C4t ..."
TAG=${1:-it}; SEL=${2:-tests/test_gpu_parity.py}; CFGS=${3:-C4q C4s C4t}
mkdir -p gpurun_out
timeout 900 python -m pytest $SEL -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
for c in $CFGS; do timeout 300 python tools/profile_one.py $c 3 2>&1 | tail -1; done | tee gpurun_out/${TAG}_times.log
