"""Timeline of c3 steps (torch.profiler / CUPTI): GPU busy time vs step time,
and the largest GPU idle gaps with the host op running at the time.

usage: python tools/c3_trace.py [config] [steps] [warmup steps]   (writes gpurun_out/<cfg>_trace.json)"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1607_04174_b200 import workloads as W  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    st = bench.setup_gpu(cfg, None, W.CONFIGS[cfg]["m"], 0)
    warm = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    for i in range(warm):
        bench.gpu_step(st, i)
    torch.cuda.synchronize()
    out = ROOT / "gpurun_out" / f"{cfg}_trace.json"
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                            torch.profiler.ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        for i in range(steps):
            with torch.profiler.record_function(f"step{i}"):
                bench.gpu_step(st, i)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    prof.export_chrome_trace(str(out))
    ev = json.load(open(out))["traceEvents"]
    kern = sorted([(e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
                   if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")])
    busy, end, gaps = 0.0, None, []
    for a, b, nm in kern:
        if end is not None and a > end:
            gaps.append((a - end, end, nm))
        if end is None or b > end:
            busy += b - max(a, end if end is not None else a)
            end = b
    span = kern[-1][1] - kern[0][0]
    print(f"{cfg}: wall {1e3 * wall / steps:.3f} ms/step, GPU span {span / 1e3 / steps:.3f} ms/step, "
          f"busy {busy / 1e3 / steps:.3f} ms/step, {len(kern) / steps:.0f} GPU ops/step")
    cpu = [(e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
           if e.get("ph") == "X" and e.get("cat") in ("cpu_op", "user_annotation", "cuda_runtime", "cuda_driver")]
    tops = {}
    for a, b, nm in kern:
        tops[nm[:60]] = tops.get(nm[:60], 0.0) + (b - a)
    for nm, t in sorted(tops.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {t / 1e3 / steps:8.3f} ms/step  {nm}")
    gaps.sort(reverse=True)
    for g, t, nm in gaps[:25]:
        host = [c[2] for c in cpu if c[0] <= t <= c[1]]
        print(f"gap {g:8.1f} us before {nm[:50]:50s} host: {host[-3:]}")


if __name__ == "__main__":
    main()
