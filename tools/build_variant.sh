#!/bin/bash
# Variant of the product library for A/B runs: recompiles bp.cu with extra
# defines and links it with the product's other objects.
#   tools/build_variant.sh OUT.so -DNAME=VALUE ...
set -eu
cd /root/repo
OUT=$1; shift
python -c "from paper_1306_5390_b200 import build; build.build()"
O=paper_1306_5390_b200/build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Iinclude \
  -Xcompiler -fPIC,-O3 "$@" -c -o /tmp/bp_variant.o paper_1306_5390_b200/csrc/bp.cu
objs=$(ls $O/*.o | grep -v '/bp.o$')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o "$OUT" $objs /tmp/bp_variant.o
echo "$OUT"
