#!/bin/bash
# On the GPU box: the round's evidence -- default bench line, the ncu launch
# list of the same command, and one ncu --set full capture of the top kernel.
#   tools/round_profile.sh TAG [workload]
set -u
TAG=${1:-r01}; WL=${2:-c4}
python bench.py --workload $WL --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_$WL.json 2> gpurun_out/bench_${TAG}_$WL.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_$WL.csv \
    python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}_$WL.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o gpurun_out/full_${TAG}_$WL \
    python bench.py --workload $WL --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_$WL.log 2>&1
