#!/bin/bash
# On the GPU box: the round's evidence -- the default bench line, the ncu
# launch list of the same command, and one ncu --set full capture of the
# fused kernel per workload (C3, C5: the five T=1 launches of one k=5 step).
#   tools/round_profile.sh TAG
set -u
TAG=${1:-r02}
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_bp -s 3 -c 1 -o gpurun_out/full_${TAG}_c4 \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_bp2 -s 15 -c 5 -o gpurun_out/full_${TAG}_c3 \
    python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_bp -s 3 -c 1 -o gpurun_out/full_${TAG}_c2 \
    python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_bp -s 15 -c 5 -o gpurun_out/full_${TAG}_c5 \
    python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_c5.log 2>&1
echo done
