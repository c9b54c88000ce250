#!/bin/bash
# Quick GPU iteration: KSG probe (C4, S=256; cell vs round-1 sweep) + the KSG parity subset.
# usage: tools/gpu_quick.sh <tag>
tag=${1:-q}
mkdir -p gpurun_out
python tools/ksg_probe.py c4 256 > gpurun_out/${tag}_probe.log 2>&1
CORR_KSG_PATH=sweep python tools/ksg_probe.py c4 256 >> gpurun_out/${tag}_probe.log 2>&1
python -m pytest tests/test_gpu_parity.py -q -x -k "ragged or large_n or invariances or dense_and_sweep or batch_equals or warp_kernel or c1_" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"
cat gpurun_out/${tag}_probe.log
tail -3 gpurun_out/${tag}_tests.log
