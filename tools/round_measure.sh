# Round measurement: bench line, kernel launch list of the same bench command (ncu, one metric,
# after the plain run exited 0), and ncu --set full of the pair kernel per C4 tiling.
# usage: bash tools/round_measure.sh r01
R=${1:-r01}
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small_$R.json 2> gpurun_out/bench_small_$R.err &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_$R.log 2>&1
for c in C4s C4t; do
  python tools/profile_one.py $c 1 > gpurun_out/full_$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_p2p_pairs -c 1 -o gpurun_out/p2p_full_$c \
      python tools/profile_one.py $c 1 >> gpurun_out/full_$c.log 2>&1
done
python tools/sample_bench.py > gpurun_out/sample_$R.jsonl 2> gpurun_out/sample_$R.err &&
ncu --set full --clock-control none --import-source on -k regex:k_sample_cells -c 3 -o gpurun_out/sample_full_$R \
    python tools/sample_bench.py 1 > gpurun_out/sample_ncu_$R.log 2>&1
