#!/bin/bash
TAG=${1:-db}; O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python -m pytest tests/test_dbscan.py -m gpu -x -q > $O/pytest_db.log 2>&1; echo rc=$? >> $O/pytest_db.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
