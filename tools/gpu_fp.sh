#!/bin/bash
TAG=${1:-fp}; O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python -m pytest tests/test_cli.py tests/test_dbscan.py -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python tools/frame_path_bench.py > $O/fp.json 2> $O/fp.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fp_launches.csv python tools/frame_path_bench.py > /dev/null 2>&1
