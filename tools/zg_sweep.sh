timeout 120 python tools/bench_zgemm.py
timeout 300 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python tools/run_eval.py c5 full 2 2>&1 | tail -2
