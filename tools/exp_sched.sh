# scheduling knobs on the C4 batch: timeline + bench value per setting
set -u
mkdir -p gpurun_out
for cfg in "FGM_TOP_SPLIT=0" "FGM_TOP_SPLIT=1" "FGM_TOP_SPLIT=2" "FGM_TOP_SPLIT=3" "FGM_TOP_SPLIT=6"; do
  echo "== $cfg"
  env $cfg python tools/timeline.py | tail -5
  for i in 1 2; do env $cfg python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"; done
done
