"""Measure streamed .rwpk save / ingest at c4 size (256^3 x K = 400, a 27 GB
file) on the GPU box: save_pack (device -> pinned blocks -> file + XXH64) and
load_pack (file -> pinned blocks -> device transpose, XXH64 from the same
bytes), GB/s of pack-file bytes, plus the peak host RSS growth (no full host
copy of the payload).  Usage: python tools/ingest_bench.py [dims] [K] [dir]."""

import json
import os
import resource
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import bench
    import paper_1607_04174_b200 as swb
    dims = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else None
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 400
    out_dir = Path(sys.argv[3]) if len(sys.argv) > 3 else Path("/tmp")
    st = bench.setup_gpu("c4", dims, m, 0)
    pack = st["pack"]
    n = st["n"]
    path = out_dir / "swb_ingest_c4.rwpk"
    rss0 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    swb.save_pack(pack, path)
    t_save = time.perf_counter() - t0
    size = path.stat().st_size
    rss1 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
    res = {"n": n, "K": m, "file_bytes": size, "save_s": t_save, "save_gbs": size / t_save / 1e9}
    for rep in range(2):   # the second read comes from the page cache
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dp = swb.load_pack(path)
        torch.cuda.synchronize()
        t_load = time.perf_counter() - t0
        res[f"load{rep}_s"] = t_load
        res[f"load{rep}_gbs"] = size / t_load / 1e9
        rows = torch.from_numpy(np.sort(np.random.default_rng(rep).choice(n, 4096, replace=False))).cuda()
        a = dp.V[rows, :m].cpu().numpy()
        b = pack.V[rows, :m].cpu().numpy().astype(np.float32).astype(np.float64)
        assert np.array_equal(a, b), "ingested basis != f32-rounded source"
        del dp
        torch.cuda.empty_cache()
    rss2 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
    res["host_rss_growth_save_MB"] = (rss1 - rss0) / 1024
    res["host_rss_growth_total_MB"] = (rss2 - rss0) / 1024
    res["payload_MB"] = 4.0 * n * m / 2 ** 20
    os.remove(path)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
