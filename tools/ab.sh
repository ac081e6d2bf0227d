#!/bin/bash
# On the GPU box: A/B of the product library against a variant build
# (interleaved runs of the default bench, parity tests on the variant).
#   tools/ab.sh paper_1306_5390_b200/libphgrms_cuda_v.so
set -u
V=${1:-paper_1306_5390_b200/libphgrms_cuda_v.so}
PHG_LIB_PATH=$PWD/$V python -m pytest tests/test_h2_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/ab_pytest.txt 2>&1
for i in 1 2 3; do
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_base_$i.json 2>/dev/null
PHG_LIB_PATH=$PWD/$V python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_var_$i.json 2>/dev/null
done
