#!/bin/bash
# One profiling pass for profiles/<round> (run on the GPU box via gpurun):
#   1. bench.py (no profiler)                                -> gpurun_out/bench.json
#   2. ncu launch list of the same bench command             -> gpurun_out/launches.csv
#   3. ncu DRAM bytes of every K3 launch of one batch solve  -> gpurun_out/sweep_dram.csv
#   4. ncu --set full of the top-level K3 launch             -> gpurun_out/sweep_top.ncu-rep
#   5. ncu --set full of the latency kernel on one 4096^2 pass -> gpurun_out/sweep_ws_c3.ncu-rep
# Each profiler pass runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"sweep|resample|upsample|coarse|stream_fill|convert" -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
python tools/prof_batch.py 256 > /dev/null || exit 1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:sweep_kernel -s 7 -c 7 --csv --log-file gpurun_out/sweep_dram.csv python tools/prof_batch.py 256 \
    > gpurun_out/ncu_dram.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 13 -c 1 \
    -o gpurun_out/sweep_top python tools/prof_batch.py 256 > gpurun_out/ncu_full.log 2>&1
python tools/prof_single.py 4096 > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:sweep_ws -s 1 -c 1 \
    -o gpurun_out/sweep_ws_c3 -f python tools/prof_single.py 4096 > gpurun_out/ncu_ws.log 2>&1
echo done
