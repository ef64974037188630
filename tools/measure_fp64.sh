# FP64 instruction counts of the P2P pair kernel and the downward kernel per config (ncu, metrics only).
# usage: bash tools/measure_fp64.sh C4q C4s C4t ...   -> gpurun_out/fp64_<cfg>.csv + gpurun_out/fp64_<cfg>.log
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
for c in "$@"; do
  python tools/profile_one.py $c 1 > gpurun_out/fp64_$c.log 2>&1 &&
  ncu --metrics $M --clock-control none -k regex:"k_p2p_pairs|k_down2" --csv --log-file gpurun_out/fp64_$c.csv \
      python tools/profile_one.py $c 1 >> gpurun_out/fp64_$c.log 2>&1
done
