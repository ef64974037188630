bash tools/measure_fp64.sh C4q C4s C4t C3 C5
for c in C4q C4s C4t C3 C5; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_p2p_pairs|k_p2p_finish" --csv --log-file gpurun_out/dram_$c.csv python tools/profile_one.py $c 1 > /dev/null 2>&1
done
ls gpurun_out
