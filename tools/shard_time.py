"""Per-rank time of a sharded evaluation, measured on ONE GPU: rank 0's shard of a config at world
size W (shard_bounds), evaluated through lg_eval_sharded with the all-reduce hook replaced by a
no-op (the only multi-GPU cost left out is that one all-reduce per evaluation: ~10 MB of raw
scalars for c4 over NVLink, tens of microseconds).  This is the device work each GPU of a W-GPU
run does, so W x (1-GPU eval time) / (this time) bounds the strong-scaling speed-up.

    python tools/shard_time.py c4 [repeats]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2304_06200_b200 import models  # noqa: E402
from paper_2304_06200_b200.costs import NativeProblem, _split  # noqa: E402
from paper_2304_06200_b200.distributed import shard_bounds  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
case = models.build_case(name)
terms, has_state = _split(case.terms)
n = case.n_states
for world in (1, 2, 4, 8):
    shard = shard_bounds(n, 0, world)
    npb = NativeProblem(case.problem, terms, case.problem.initial_state if has_state else None, case.problem.basis,
                        shard=shard)
    buf = torch.zeros(npb.raw_size(case.field.n_steps), dtype=torch.float64, device="cuda:0")
    npb.set_raw_buffer(buf.data_ptr(), buf.numel())
    npb.set_stream(torch.cuda.current_stream().cuda_stream)
    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        npb.grad_sharded(case.field, lambda ptr, count: 0)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name} world={world} shard={shard} ({shard[1] - shard[0]} trajectories) engine={npb.engine}: "
          f"{1e3 * min(ts[1:]):.1f} ms per evaluation on rank 0", flush=True)
    del npb, buf
