# Round checkpoint on one B200: the whole -m gpu suite, the driver's exact bench command, bench
# lines of the other workloads, the kernel launch list of the bench command (ncu, one metric,
# after the plain run exited 0) and ncu --set full of the pair kernel on C4t.
# usage: bash tools/checkpoint.sh TAG
T=${1:-ck}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_$T.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_$T.log
python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver_$T.json 2> gpurun_out/bench_driver_$T.err; echo "bench rc=$?"
for w in C3 C5 C2 C1; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${w}_$T.json 2> gpurun_out/bench_${w}_$T.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_p2p_pairs -c 1 -o gpurun_out/p2p_full_C4t_$T \
    python tools/profile_one.py C4t 1 > gpurun_out/p2p_full_C4t_$T.log 2>&1
echo done
