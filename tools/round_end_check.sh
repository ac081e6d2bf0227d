bash tools/ab_c3.sh b2late
bash tools/final_check.sh
python bench.py --impl reference > gpurun_out/fc_bench_ref.json 2>gpurun_out/fc_bench_ref.err
for wl in c2 c5; do python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/fc_$wl.json 2>/dev/null; done
