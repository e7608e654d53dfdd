timeout 300 python tools/fused_check.py --var RVK_PREP_SCORE --a 1 --b 0
for v in 1 0; do for c in 4; do for T in 256 1024; do echo "== prep_score=$v config $c T=$T"; RVK_PREP_SCORE=$v timeout 300 python bench.py --config $c --max-trials $T --no-cpu-baseline --e2e-steps 4 --latency-reps 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('value %.3e ms %.3f frac %.3f stages %s lat %.3f'%(d['value'],d['ms_per_step'],r['frac'],{k:round(v,3) for k,v in r['stage_ms_per_step'].items()},d['p50_frame_latency_ms']))"; done; done; done
RVK_PREP_SCORE=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:"fused_warp|select_warp" -c 2 -o gpurun_out/r2_ps python tools/one_call.py --config 4 --frames 16 --reps 1 > /dev/null 2>&1
