# end-of-round extras on one B200: per-launch time + DRAM traffic of one step per config, ncu --set
# full of the leaf-level M2L (C4t), multi-rank projections (C4, C5)
# usage: bash tools/round_final.sh TAG
T=${1:-final}
mkdir -p gpurun_out
for c in C4q C4s C4t C3 C5; do
  python tools/profile_one.py $c 1 > gpurun_out/tab_$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/tab_$c.csv python tools/profile_one.py $c 1 >> gpurun_out/tab_$c.log 2>&1
  python tools/ncu_table.py gpurun_out/tab_$c.csv > gpurun_out/launch_dram_table_${c}_$T.txt 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_down_mma --launch-skip 8 -c 1 \
    -o gpurun_out/m2l_leaf_C4t_$T python tools/profile_one.py C4t 1 > gpurun_out/m2l_leaf_C4t_$T.log 2>&1
python tools/multirank_project.py --workload C4 --ranks 1,2,4,8 --reps 3 > gpurun_out/multirank_projection_C4_$T.json 2> gpurun_out/mrp_C4.err
python tools/multirank_project.py --workload C5 --ranks 1,8 --reps 2 > gpurun_out/multirank_projection_C5_$T.json 2> gpurun_out/mrp_C5.err
echo done
