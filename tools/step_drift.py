"""Per-step device time over a long run of one config (CUDA events between
steps, no syncs inside), printed as averages over blocks of 10 steps: shows
whether a step's cost drifts with the step count.

usage: python tools/step_drift.py [config] [steps]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1607_04174_b200 import workloads as W  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 150
    st = bench.setup_gpu(cfg, None, W.CONFIGS[cfg]["m"], 0)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    import gc
    import os
    do_gc = os.environ.get("DRIFT_GC") == "1"
    mem = []
    ev[0].record()
    for i in range(steps):
        bench.gpu_step(st, i)
        ev[i + 1].record()
        if do_gc:
            gc.collect()
        if i % 10 == 9:
            mem.append((torch.cuda.memory_allocated() / 1e9, torch.cuda.memory_reserved() / 1e9, len(gc.get_objects())))
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    for b in range(0, steps, 10):
        blk = ms[b:b + 10]
        a, r, o = mem[b // 10] if b // 10 < len(mem) else (0, 0, 0)
        print(f"steps {b:4d}-{b + len(blk) - 1:4d}: {sum(blk) / len(blk):8.3f} ms  alloc {a:.1f} GB reserved {r:.1f} GB "
              f"objs {o} "
              f"[{' '.join(f'{x:.2f}' for x in blk)}]")


if __name__ == "__main__":
    main()
