timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_pytest.log 2>&1; tail -3 gpurun_out/r2k_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/bench_all.sh r2k > /dev/null 2>&1
python tools/summarize_bench.py gpurun_out/r2k_*.json
bash tools/profile_r2.sh > /dev/null 2>&1; ls gpurun_out | grep r2_c
