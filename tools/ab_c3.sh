mkdir -p gpurun_out
python -m pytest tests/test_h2b2_gpu.py tests/test_h2_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/ab2_pytest.txt 2>&1
for i in 1 2 3; do
PHG_LIB_PATH=$PWD/paper_1306_5390_b200/libphgrms_cuda_base.so python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab2_base_c3_$i.json 2>/dev/null
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab2_var_c3_$i.json 2>/dev/null
done
for wl in c2 c5; do python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/ab2_var_$wl.json 2>gpurun_out/ab2_var_$wl.err; done
tail -2 gpurun_out/ab2_pytest.txt
