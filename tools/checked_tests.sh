#!/bin/bash
# The checked build (-DLT_CHECKS: device asserts on every derived index,
# stack depth and queue slot in the hot kernels) under the whole -m gpu
# suite and smoke(): the in-house substitute for compute-sanitizer, which
# this GPU pool does not allow.  Any failed assert aborts the kernel and
# fails the test that launched it.
mkdir -p gpurun_out
python -c "from paper_2407_19977_b200.build import build; build(variant='checks', defines=('LT_CHECKS',))"
export LUXB200_LIB=$PWD/paper_2407_19977_b200/_build/variant_checks/libluxb200.so
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/checked_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/checked_smoke.log
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/checked_gputests.log
