# bench (+ optional env) per library variant (FGMATTE_B200_LIB)
set -u
mkdir -p gpurun_out
for v in paper_2006_14970_b200/libfgmatte_b200.so "$@"; do
  echo "== $v"
  for i in 1 2; do FGM_PYRAMID_MAIN=1 FGMATTE_B200_LIB=$PWD/$v python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench(pyr main)', round(d['value']), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"; done
  FGMATTE_B200_LIB=$PWD/$v python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
done
