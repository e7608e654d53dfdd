# Round-2 final validation on the GPU box (repo root): the -m gpu suite, the
# fuzz parity sweeps over every kernel path.
# Outputs under gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/vf_pytest.log 2>&1; echo "rc $?" >> gpurun_out/vf_pytest.log
F=gpurun_out/vf_fuzz.txt; : > $F
for env in "" "RVK_PREP_SCORE=1" "RVK_FUSED=1" "RVK_PREP_SCORE=0 RVK_FUSED=0"; do
  echo "== $env" >> $F; env $env timeout 600 python tools/fuzz_parity.py --frames 10000 --seed 7 2>&1 | tail -1 >> $F
done
for env in "" "RVK_PREP_SCORE=1"; do
  echo "== stress $env" >> $F; env $env timeout 600 python tools/fuzz_parity.py --stress --frames 1000 --seed 7 2>&1 | tail -1 >> $F
done
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck over tools/sanitize.py)
# is closed on the GPU pool since this round's last capture (profiles/r2_sanitizer.txt).
