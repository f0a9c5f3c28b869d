"""c3 select_m timing: per interaction round, select_m on the current pack
(CUDA events around the call, host sync included as the API has it), the
decision, and the step's own update_and_solve time.  Run it under
`ncu --metrics gpu__time_duration.sum` for the per-kernel split.

usage: python tools/select_bench.py [reps]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1607_04174_b200 as swb  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    st = bench.setup_gpu("c3", None, 150, 0)
    pol = swb.AdaptivePolicy(epsilon=st["params"]["epsilon"])
    pack = st["pack"]
    for r, prob in enumerate(st["round_probs"]):
        for _ in range(2):
            swb.select_m(pack, prob, pol)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            m, info = swb.select_m(pack, prob, pol)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"round {r}: S={prob.seeds.n_seeds} m_use={m} steps={len(info['steps'])} "
              f"select_m {1e3 * min(ts):.3f} ms (min of {reps}), median {1e3 * sorted(ts)[len(ts) // 2]:.3f}",
              flush=True)


if __name__ == "__main__":
    main()
