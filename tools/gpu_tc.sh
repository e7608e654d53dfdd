#!/bin/bash
# TC iteration: smoke + gpu tests + bench (tc and ffma) + launch list
TAG=${1:-tc}; O=gpurun_out/$TAG; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench.json 2> $O/bench.err
for c in 3 4; do timeout 300 python bench.py --config $c --no-cpu-baseline --steps 50 --e2e-steps 10 > $O/bench_c$c.json 2>> $O/bench.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score|prep|select" -c 30 --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --streams 1 --e2e-steps 2 > /dev/null 2>&1
