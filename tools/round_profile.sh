#!/bin/bash
# On the GPU box: the round's evidence -- the bench lines of every workload
# and the reference arm, the ncu launch list of the default command, one
# ncu --set full capture of the fused kernel per workload (C3, C5: the five
# single-buffer T=1 launches of one k=5 step), and the side-op lines.
#   tools/round_profile.sh TAG [PART]   PART: all (default), lines, ncu12, ncu3, ncu5
# (gpurun brings back at most 64 MiB: the full captures go in separate calls)
set -u
TAG=${1:-r02}
PART=${2:-all}
O=gpurun_out
if [ "$PART" = all ] || [ "$PART" = lines ]; then
python bench.py --steps 20 --warmup 5 > $O/bench_${TAG}_c4.json 2> $O/bench_${TAG}_c4.err
for w in c1 c2; do python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${TAG}_$w.json 2>/dev/null; done
for w in c3 c5; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${TAG}_$w.json 2>/dev/null; done
python bench.py --workload c5 --k 10 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${TAG}_c5_k10.json 2>/dev/null
python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_${TAG}_ref.json 2>/dev/null
python bench_ops.py > $O/bench_ops_${TAG}.jsonl 2>/dev/null
fi
if [ "$PART" = all ] || [ "$PART" = ncu12 ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_${TAG}_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_${TAG}_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_bp -s 3 -c 1 -o $O/full_${TAG}_c4 \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_${TAG}_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_bp -s 3 -c 1 -o $O/full_${TAG}_c2 \
    python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_${TAG}_c2.log 2>&1
fi
if [ "$PART" = all ] || [ "$PART" = ncu3 ]; then
ncu --set full --clock-control none --import-source on -k regex:fused_bp2 -s 15 -c 5 -o $O/full_${TAG}_c3 \
    python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_${TAG}_c3.log 2>&1
fi
if [ "$PART" = all ] || [ "$PART" = ncu5 ]; then
ncu --set full --clock-control none --import-source on -k regex:fused_bp -s 15 -c 5 -o $O/full_${TAG}_c5 \
    python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_${TAG}_c5.log 2>&1
fi
echo done
