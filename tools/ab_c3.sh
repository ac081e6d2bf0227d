#!/bin/bash
# On the GPU box: interleaved C3 (beta=2) runs of the product library and
# variant builds, beta=2 parity tests on each variant.
#   tools/ab_c3.sh TAG1 TAG2 ...   (paper_1306_5390_b200/libphgrms_cuda_TAG.so)
set -u
mkdir -p gpurun_out
for v in "$@"; do
PHG_LIB_PATH=$PWD/paper_1306_5390_b200/libphgrms_cuda_$v.so python -m pytest tests/test_h2b2_gpu.py -x -q > gpurun_out/ab3_pytest_$v.txt 2>&1
done
for i in 1 2 3; do
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab3_base_$i.json 2>/dev/null
for v in "$@"; do
PHG_LIB_PATH=$PWD/paper_1306_5390_b200/libphgrms_cuda_$v.so python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab3_${v}_$i.json 2>/dev/null
done
done
tail -qn1 gpurun_out/ab3_pytest_*.txt
