#!/bin/bash
# On the GPU box: product GPU tests + smoke, A/B against a variant library,
# and the round's C4 evidence (bench line, launch list, ncu --set full).
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/fc_gputests.log 2>&1; echo TESTS_RC=$? >> gpurun_out/fc_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo SMOKE_RC=$? >> gpurun_out/fc_smoke.log
if [ -f paper_1306_5390_b200/libphgrms_cuda_v.so ]; then bash tools/ab.sh paper_1306_5390_b200/libphgrms_cuda_v.so; fi
bash tools/round_profile.sh r01c c4
tail -2 gpurun_out/fc_gputests.log; tail -1 gpurun_out/fc_smoke.log
