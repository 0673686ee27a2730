timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 120 python tools/run_eval.py c3 full 3 2>&1 | tail -2
timeout 200 python tools/run_eval.py c4 400 2 2>&1 | tail -2
TAG=default timeout 300 python tools/racecheck.py 30
