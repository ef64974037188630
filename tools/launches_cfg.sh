# Launch list (one metric, serialised) of one build + evaluate per config; run after the same
# profile_one command exited 0.   usage: bash tools/launches_cfg.sh C4q C4s C4t
for c in "$@"; do
  python tools/profile_one.py $c 1 > gpurun_out/lc_$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lc_$c.csv \
      python tools/profile_one.py $c 1 >> gpurun_out/lc_$c.log 2>&1
done
