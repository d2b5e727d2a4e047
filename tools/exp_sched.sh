# scheduling knobs on the C4 batch: timeline + bench value per setting
set -u
mkdir -p gpurun_out
for cfg in "FGM_SMALL_WPS=0:0" "FGM_SMALL_WPS=4:8" "FGM_SMALL_WPS=4:8 FGM_SIDE_BLOCKS_RT=0" "FGM_SMALL_WPS=2:8 FGM_SIDE_BLOCKS_RT=0" "FGM_SMALL_WPS=4:8 FGM_SIDE_BLOCKS_RT=8"; do
  echo "== $cfg"
  env $cfg python tools/timeline.py
  for i in 1 2; do env $cfg python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"; done
done
