timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python tools/run_eval.py c1 full 3 2>&1 | tail -2
timeout 120 python tools/run_eval.py c2 full 5 2>&1 | tail -2
