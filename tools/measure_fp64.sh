# FP64 work of the hot kernels under ncu (metrics only, --clock-control none):
#  * the one-pair-per-thread math microbenchmark (tools/fpair_micro.py) -> F_pair
#  * k_p2p_pairs and k_down_mma (M2L + L2L on DMMA) per config
# usage: bash tools/measure_fp64.sh C4q C4s C4t ...   -> gpurun_out/fp64_<cfg>.{csv,log}
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
python tools/fpair_micro.py > gpurun_out/fp64_micro.log 2>&1 &&
ncu --metrics $M --clock-control none -k regex:k_debug_p2p_math --csv --log-file gpurun_out/fp64_micro.csv \
    python tools/fpair_micro.py >> gpurun_out/fp64_micro.log 2>&1
for c in "$@"; do
  python tools/profile_one.py $c 1 > gpurun_out/fp64_$c.log 2>&1 &&
  ncu --metrics $M --clock-control none -k regex:"k_p2p_pairs|k_down_mma" --csv --log-file gpurun_out/fp64_$c.csv \
      python tools/profile_one.py $c 1 >> gpurun_out/fp64_$c.log 2>&1
done
