#!/bin/bash
# Build the chaos variant (random pauses before publishes/polls/barrier waits) and run the GPU
# suite against it.  Usage (box): bash tools/chaos.sh TAG   (build it here first:
# tools/build_variant.sh chaos -DGCM_CHAOS)
tag=${1:-r02}
out=gpurun_out/${tag}_chaos; mkdir -p $out
GCM_LIB_PATH=$PWD/paper_1011_1173_b200/lib/variants/libgcm_chaos.so timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1
echo "chaos pytest rc=$?" | tee -a $out/pytest.log
tail -3 $out/pytest.log
