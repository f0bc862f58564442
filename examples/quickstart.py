"""Quickstart (README): 512 independent Sep-CMA-ES runs on 1000-D Rastrigin, 100 generations,
through the Python binding of the C ABI (the paper's Listing 1 ask–evaluate–tell loop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2212_04180_b200 import strategy as S  # noqa: E402

es = S.Strategy(W.SEP_CMA_ES, 256, 1000,
                [W.run_params(W.SEP_CMA_ES, seed, init_min=-5.12, init_max=5.12) for seed in range(512)])
for gen in range(100):
    x = es.ask()                       # [R, N, D] on the GPU
    f = es.eval(W.RASTRIGIN, x)        # or any fitness of your own, [R, N]
    es.tell(f)                         # regenerates the noise from the counter; x is not re-read
best = es.get("best_f")
print(f"best fitness over 512 runs after 100 generations: min {best.min().item():.2f}, "
      f"median {best.median().item():.2f}")
es.close()
