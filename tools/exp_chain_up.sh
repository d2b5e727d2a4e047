set -u
mkdir -p gpurun_out
for wps in 9 6 3; do echo "warps/SM=$wps"; FGM_SWEEP_WARPS_PER_SM=$wps python tools/time_configs.py 3 5; done > gpurun_out/chain_exp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:upsample_kernel -s 7 -c 7 -o gpurun_out/up_full python tools/prof_batch.py 256 > gpurun_out/ncu_up.log 2>&1
echo done
