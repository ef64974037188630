# ncu --set full (with source) of one launch of a kernel in one build + evaluate of a config
# usage: bash tools/ncu_kernel.sh CFG KERNEL_REGEX TAG [launch-skip]
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip ${4:-0} -c 1 \
    -o gpurun_out/$3 python tools/profile_one.py $1 1 > gpurun_out/$3.log 2>&1
