run() { echo "== $*"; env "$@" timeout 300 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 4 $EXTRA 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('value %.3e ms %.3f score_frac %.3f stages %s'%(d['value'],d['ms_per_step'],r['frac'],{k:round(v,3) for k,v in r['stage_ms_per_step'].items()}))"; }
run RVK_FUSED=1
run RVK_FUSED=0
run RVK_FUSED=0 RVK_SCORE_CTAS=2
EXTRA="--streams 3" run RVK_FUSED=0 RVK_SCORE_CTAS=2
EXTRA="--streams 3" run RVK_FUSED=0 RVK_SCORE_CTAS=1
EXTRA="--streams 3" run RVK_FUSED=0
