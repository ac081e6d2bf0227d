#!/bin/bash
# Dev loop: rebuild the CUDA library, then on a B200 run the GPU tests, the
# default bench and one ncu --set full capture of the fused kernel.
#   tools/gpu_iter.sh TAG [kernel-regex] [extra env for the bench]
set -u
cd /root/repo
TAG=${1:-dev}; KRE=${2:-fused_h2}; ENVS=${3:-}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude \
  -o /tmp/lib_iter.so paper_1306_5390_b200/csrc/phgrms_cuda.cu 2>&1 | grep -E "error" && exit 1
cp /tmp/lib_iter.so paper_1306_5390_b200/libphgrms_cuda.so
timeout 2400 /usr/local/graft/bin/gpurun --timeout 900 -- "python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; $ENVS python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; $ENVS ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o gpurun_out/$TAG python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1" > /tmp/gpurun_$TAG.log 2>&1
tail -1 /tmp/gpurun_$TAG.log
tail -2 gpurun_out/pytest_gpu.txt
python -c "
import json
d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1]); print('value', d['value'], 'kernel_ms', d['roofline']['kernel_ms'], 'e2e', d['e2e']['value'])
"
