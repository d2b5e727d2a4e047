#!/bin/bash
# One K3 development iteration on the GPU box: parity subset, batch timeline,
# config timings, and (if those pass) an ncu capture of the top-level sweep.
#   gpurun -- bash tools/iter.sh <tag>
set -u
tag=${1:-it}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "sweep_passes or border_modes or ml_vs_oracle_shapes or per_level or k4_throughput or random_sizes" > gpurun_out/${tag}_par.log 2>&1
rc=$?
echo "parity rc $rc" >> gpurun_out/${tag}_par.log
tail -3 gpurun_out/${tag}_par.log
[ $rc -ne 0 ] && exit 1
timeout 200 python tools/timeline.py 256 > gpurun_out/${tag}_timeline.txt 2>&1 || exit 1
tail -4 gpurun_out/${tag}_timeline.txt
timeout 300 python tools/time_configs.py > gpurun_out/${tag}_configs.txt 2>&1
cat gpurun_out/${tag}_configs.txt
if [ "${NCU:-1}" = "1" ]; then
  python tools/prof_batch.py 256 > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 6 -c 1 \
      -o gpurun_out/${tag}_sweep python tools/prof_batch.py 256 > gpurun_out/${tag}_ncu.log 2>&1
  tail -1 gpurun_out/${tag}_ncu.log
fi
