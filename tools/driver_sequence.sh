set -o pipefail
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02e.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r02e.log
timeout 900 python bench.py > gpurun_out/bench_default_r02e.json 2> gpurun_out/bench_default_r02e.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02e.json 2> gpurun_out/bench_ref_r02e.err; echo "ref rc=$?"
cat gpurun_out/bench_ref_r02e.json | cut -c1-600
