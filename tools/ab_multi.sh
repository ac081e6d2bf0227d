#!/bin/bash
# On the GPU box: interleaved C4 runs of the product library and variant
# builds, parity tests on each variant.
#   tools/ab_multi.sh TAG1 TAG2 ...   (paper_1306_5390_b200/libphgrms_cuda_TAG.so)
set -u
mkdir -p gpurun_out
for v in "$@"; do
PHG_LIB_PATH=$PWD/paper_1306_5390_b200/libphgrms_cuda_$v.so python -m pytest tests/test_h2_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/abm_pytest_$v.txt 2>&1
done
python -m pytest tests/test_h2_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/abm_pytest_base.txt 2>&1
for i in 1 2 3; do
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/abm_base_$i.json 2>/dev/null
for v in "$@"; do
PHG_LIB_PATH=$PWD/paper_1306_5390_b200/libphgrms_cuda_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/abm_${v}_$i.json 2>/dev/null
done
done
for wl in c2 c5; do python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/abm_base_$wl.json 2>/dev/null; done
tail -qn1 gpurun_out/abm_pytest_*.txt
