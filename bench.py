"""Benchmark of the online hot path on B200 (one JSON line on rank 0).

One *step* = one interaction of the BASELINE config-4 workload (256^3 volume,
K = 400 eigenvectors, V = 54 GB FP64 resident in HBM):
  1. first-order basis update for beta 80 -> 110 (alternating 110 -> 80 on
     odd steps so every step is a valid update of the previous one):
     graph coefficients, difference stencil dL V, DMMA symmetric projection
     P = V^T dL V, refresh eigenvalues + gap-guarded coefficients C,
     DMMA rotation V' = V C;
  2. 4-label reduced-basis random-walker solve with 200 seeds per label
     (gamma = 0): seed projections, (S+1)^2 LU + rcond, reconstruction +
     finalize + per-voxel argmax.
value = N*K / step time (whole job, all ranks).  e2e = the same through the
public API with host seeds in and host labels out every step.

--impl reference times the reference algorithm's CPU restatement
(oracle/rw_oracle.py, numpy/scipy on all host cores) on a bounded z-slab
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os

# with SWB_EMIT=1 the c4 step keeps two 54 GB bases and the rotation's 46 GB
# of digit planes resident; expandable segments keep the allocator's freed
# setup temporaries from fragmenting HBM around them
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


METRIC = "basis-update N·K/s and RW-solve voxels/s; % HBM / FP64-tensor roofline"
UNIT = "N·K/s"
CPU_SLAB_PLANES = 4          # the --impl reference arm's per-step sample (K steps must end in minutes)
CPU_SLAB_PLANES_ALL = 32     # the all-cores cpu_baseline sample (a 256x256x32 z-slab)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 6 at c4; small configs run enough steps for ~1.5 s of timed "
                         "region, so the clock sampler sees the load)")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c4")
    ap.add_argument("--dims", default=None, help="override volume dims, e.g. 64,64,64")
    ap.add_argument("--m", type=int, default=None, help="override K")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="time CUDA-graph replays of the step (two chained steps per graph; fixed seeds)")
    ap.add_argument("--profile-steps", type=int, default=0, help="ncu helper: run N steps, no timing")
    ap.add_argument("--sharded", action="store_true", help="use the z-slab sharded path even at N=1")
    ap.add_argument("--method", choices=["first_order", "rayleigh"], default="first_order",
                    help="basis update of each step: the north-star first-order update (default) or the "
                         "reference's eigenvalue-only refresh (refresh.py:63-82)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, interval_ms: int = int(os.environ.get("SWB_SMI_MS", "200"))):
        self.index = index
        self.interval_ms = interval_ms
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.interval_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 5.0):
        """Block until nvidia-smi has produced its first sample, so its
        start-up (NVML init, driver queries) happens before the timed region
        rather than inside its first step."""
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.05)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement on a bounded z-slab sample
# ---------------------------------------------------------------------------

def cpu_sample(cfg: str, dims, m: int, planes: int = CPU_SLAB_PLANES):
    from paper_1607_04174_b200 import workloads as W
    w = W.make_image(cfg, dims)
    d3 = len(w.dims) == 3
    sdims = (w.dims[0], w.dims[1], planes) if d3 else w.dims
    n = int(np.prod(sdims))
    z0 = 0
    if d3:  # the slab window that sees the most labelled objects
        plane = w.dims[0] * w.dims[1]
        t3 = w.truth.reshape(w.dims[2], plane)
        best = (-1, -1)
        for z in range(0, w.dims[2] - planes + 1):
            win = t3[z:z + planes]
            score = (len(np.unique(win[win >= 0])), int((win >= 0).sum()))
            if score > best:
                best, z0 = score, z
        z0 *= plane
    img = w.intensities[z0:z0 + n]
    truth = w.truth[z0:z0 + n]
    moving = w.params["moving"][z0:z0 + n] if "moving" in w.params else None
    rng = np.random.default_rng([W.CFG_INDEX[cfg], 9])
    G = rng.standard_normal((n, m))
    for _ in range(2):  # CholeskyQR2
        R = np.linalg.cholesky(G.T @ G).T
        G = np.linalg.solve(R.T, G.T).T
    lam = W.synthetic_lambda(cfg, m)
    seeds, labs = W.sample_region_seeds(truth, w.params["labels"], w.params["seeds_per_label"], rng)
    cut = W.cut_for(w) if not d3 else None
    return dict(dims=sdims, img=img, V=np.asfortranarray(G), lam=lam, seeds=seeds, labs=labs, n=n,
                params=w.params, moving=moving, cut=cut[1:] if cut is not None else None)


def cpu_step(s, beta0, beta1, labels):
    from oracle import rw_oracle as O
    p = s["params"]
    lap0 = O.build_laplacian(s["img"], s["dims"], beta0, p["weight_mode"], p["connectivity"])
    cut = None
    if s.get("cut") is not None:   # c2: the block-boundary edge cut (the GPU arm's topology update)
        x0, y0 = s["cut"]
        cut = O.block_cut_mask(s["dims"], x0, y0, size=p["cut_block"], connectivity=p["connectivity"])
    lap1 = O.build_laplacian(s["img"], s["dims"], beta1, p["weight_mode"], p["connectivity"], cut_edges=cut)
    V1, lam1, _, _, _ = O.first_order_update(s["V"], s["lam"], lap0, lap1)
    if s["moving"] is not None:  # c5: registration data term + gamma > 0 solve + expected displacement
        vec = O.grid_vectors(p["grid"])
        pri, _ = O.similarity_priors(s["img"], s["moving"], s["dims"], vec, p["patch_radius"])
        u = O.solve_fast(V1, lam1, lap1.d_sqrt, lap1.matrix, [], [], labels, gamma=p["gamma"], priors=pri)
        return O.hard_labels(u), u @ vec
    m_use = None
    if p.get("epsilon") is not None:   # c3: K from the accuracy target (adaptive.py:133-185)
        m_use, _ = O.select_m(V1, lap1.d_sqrt, s["seeds"], s["labs"], labels, epsilon=p["epsilon"])
    u = O.solve_fast(V1, lam1, lap1.d_sqrt, lap1.matrix, s["seeds"], s["labs"], labels, m_use=m_use)
    return O.hard_labels(u)


def cpu_model() -> str:
    """The host CPU's model name (lscpu, else /proc/cpuinfo)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def blas_threads() -> int:
    from threadpoolctl import threadpool_info
    info = threadpool_info()
    return max([int(x.get("num_threads", 1)) for x in info] or [1])


def _time_cpu(s, threads, steps):
    """Best of ``steps`` oracle steps under a BLAS thread limit (None = all)."""
    from threadpoolctl import threadpool_limits
    p = s["params"]
    t = []
    # None = every host core, stated explicitly: torchrun exports OMP_NUM_THREADS=1
    with threadpool_limits(limits=threads or os.cpu_count()):
        used = blas_threads()
        for i in range(steps):
            b0, b1 = (p["beta0"], p["beta1"]) if i % 2 == 0 else (p["beta1"], p["beta0"])
            t0 = time.perf_counter()
            cpu_step(s, b0, b1, p["labels"])
            t.append(time.perf_counter() - t0)
    return min(t), used


def _describe(cfg, s, m):
    what = ("priors + gamma=1 solve + labels + displacement" if cfg == "c5" else
            "select_m + gamma=0 solve + labels" if s["params"].get("epsilon") is not None else
            "gamma=0 solve + labels")
    where = f"z-slab {'x'.join(map(str, s['dims']))}" if len(s["dims"]) == 3 else f"{'x'.join(map(str, s['dims']))}"
    return f"{cfg} {where} ({s['n']} voxels) x K={m}: oracle first-order update + {what}"


def cpu_baseline(cfg, dims, m):
    """The oracle restatement (oracle/rw_oracle.py on numpy/scipy/OpenBLAS) on
    the box's host cores: all cores on a 32-plane z-slab of a
    3-D volume (the whole image in 2-D) and 1 thread on the 4-plane slab,
    both reported as N·K/s; the per-N·K rate is extrapolated linearly in N to
    the full volume (the oracle's work is linear in N: measured 22.6 vs 22.9
    M N·K/s at 4 vs 8 planes).  The scipy-sparse parts are single-threaded
    whatever the limit."""
    d3 = len(W_dims(cfg, dims)) == 3
    small = cpu_sample(cfg, dims, m, planes=CPU_SLAB_PLANES)
    big = cpu_sample(cfg, dims, m, planes=CPU_SLAB_PLANES_ALL) if d3 else small
    _time_cpu(small, None, 1)                            # warm-up: imports, BLAS thread pool
    steps = 1 if d3 else 2
    t_all, th_all = _time_cpu(big, None, steps)
    t_one, _ = _time_cpu(small, 1, steps)
    v_all = big["n"] * m / t_all
    v_one = small["n"] * m / t_one
    return {"value": v_all, "unit": UNIT, "cores": th_all, "kind": "port",
            "sample": f"{_describe(cfg, big, m)}; all {th_all} BLAS threads, best of {steps}, {t_all:.2f} s/step",
            "extrapolated": d3, "extrapolation": "per-N·K rate of the slab, linear in N" if d3 else None,
            "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
            "all_cores": {"value": v_all, "threads": th_all, "s_per_step": t_all, "voxels": big["n"]},
            "single_thread": {"value": v_one, "threads": 1, "s_per_step": t_one, "voxels": small["n"],
                              "sample": f"{_describe(cfg, small, m)}; 1 BLAS thread (threadpoolctl), best of "
                                        f"{steps}"}}


def W_dims(cfg, dims):
    from paper_1607_04174_b200 import workloads as W
    return tuple(dims) if dims else tuple(W.CONFIGS[cfg]["dims"])


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1607_04174_b200 import workloads as W
    cfg = args.config
    dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
    m = args.m or W.CONFIGS[cfg]["m"]
    s = cpu_sample(cfg, dims, m)
    p = s["params"]
    # all the host threads, also under torchrun (which exports OMP_NUM_THREADS=1 to every rank)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=os.cpu_count()):
        threads = blas_threads()
        for i in range(args.warmup):
            cpu_step(s, p["beta0"], p["beta1"], p["labels"])
        t0 = time.perf_counter()
        for i in range(args.steps):
            b0, b1 = (p["beta0"], p["beta1"]) if i % 2 == 0 else (p["beta1"], p["beta0"])
            cpu_step(s, b0, b1, p["labels"])
        sec = (time.perf_counter() - t0) / max(args.steps, 1)
    value = s["n"] * m / sec
    dims_full = dims or W.CONFIGS[cfg]["dims"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg} {'x'.join(map(str, dims_full))} K={m}", "K": m,
                       "sample_voxels": s["n"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{_describe(cfg, s, m)}; oracle/rw_oracle.py on numpy/scipy/OpenBLAS, all "
                                       f"{threads} BLAS threads, mean of {args.steps} steps after {args.warmup}",
                             "extrapolated": len(s["dims"]) == 3,
                             "extrapolation": "per-N·K rate of the slab, linear in N" if len(s["dims"]) == 3
                             else None, "cpu_model": cpu_model(), "host_cpus": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def setup_gpu(cfg, dims, m, rank):
    import torch

    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import workloads as W
    from paper_1607_04174_b200.device import DevicePack, LatticeSpec, round_up
    w = W.make_image(cfg, dims)
    p = w.params
    n = int(np.prod(w.dims))
    image = swb.Image(w.dims, w.intensities)
    lattice = LatticeSpec.make(w.dims, p["connectivity"], p["weight_mode"])
    V = W.orthonormal_basis_device(n, m, seed=W.CFG_INDEX[cfg] * 1000 + 17 + rank)
    lam = torch.from_numpy(W.synthetic_lambda(cfg, m)).cuda()
    img_dev = torch.from_numpy(np.array(w.intensities)).cuda()
    g0 = swb.DeviceGraph.build(img_dev, lattice, p["beta0"])
    prov = swb.PackProvenance(image_hash=image.content_hash())
    pack = DevicePack(V, m, lam, g0.d_sqrt_dev, g0.dnorm, w.dims, (), p["beta0"], prov, lattice,
                      image_dev=img_dev, graph=g0)
    # the API caches the device copy of the image per Image object
    from paper_1607_04174_b200 import api
    api._image_entry(image)[2] = img_dev
    if cfg == "c5":
        from paper_1607_04174_b200 import registration as R
        moving = swb.Image(w.dims, p["moving"])
        return dict(w=w, image=image, moving=moving, grid=R.DisplacementGrid(p["grid"]), pack=pack, prob=None, n=n,
                    m=m, params=p, seeds_n=0)
    seeds, labs = W.seeds_for(w)
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(n, seeds, labs))
    cut = W.cut_for(w)
    round_probs = None
    if p.get("rounds"):   # c3: cumulative seeds of rounds 0..r (union, first label wins)
        round_probs, acc_i, acc_l = [], np.empty(0, np.int64), np.empty(0, np.int64)
        for r in range(p["rounds"]):
            si, sl = W.seeds_for(w, r)
            acc_i, first = np.unique(np.concatenate([acc_i, si]), return_index=True)
            acc_l = np.concatenate([acc_l, sl])[first]
            round_probs.append(swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(n, acc_i, acc_l)))
    return dict(w=w, image=image, pack=pack, prob=prob, n=n, m=m, params=p, seeds_n=len(seeds),
                cut=torch.from_numpy(cut[0]).cuda() if cut is not None else None, round_probs=round_probs)


def _next_pack(state, beta, i=0):
    """Chained update in ping-pong mode: V' goes into the previous step's
    (retired) basis buffer, so no 54 GB allocation happens per step.  A
    cut-edge config (c2) removes the block-boundary edges on even steps and
    restores them on odd steps (beta unchanged), so every step is a real
    topology update of the previous pack."""
    import paper_1607_04174_b200 as swb
    if state.get("method") == "rayleigh":
        # the reference's refresh: new eigenvalues + column order on the
        # resident basis (no rotation, nothing to ping-pong)
        base = state.setdefault("base", state["pack"])
        pack = swb.refresh(base, state["image"], beta)
        state["pack"] = pack
        return pack
    if state["params"].get("epsilon") is not None:   # c3: from the precomputed pack (_next_pack_and_solve)
        base = state.setdefault("base", state["pack"])
        pack = swb.update_basis(base, state["image"], state["params"]["beta1"], method="first_order",
                                out=state.get("spare"))
        state["spare"] = pack.V
        state["pack"] = pack
        return pack
    spare = state.pop("spare", None)
    old = state["pack"]
    cut = state.get("cut") if i % 2 == 0 else None
    pack = swb.update_basis(old, state["image"], beta, cut_edges=cut, method="first_order", out=spare)
    state["spare"] = old.V
    state["pack"] = pack
    return pack


def registration_solve(state, pack, fixed, moving):
    """c5: data term -> 125-label gamma > 0 solve -> expected displacement,
    all on the device (registration.py:153-229, fast branch)."""
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import registration as R
    p = state["params"]
    pri = R.similarity_priors(fixed, moving, state["grid"], p["patch_radius"])
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(state["n"], [], []),
                            priors=pri.values_dev, gamma=p["gamma"])
    field = swb.solve_fast(pack, pack.laplacian, prob)
    field.displacement_dev = R.expected_displacement_device(field, state["grid"])
    return field


def _adaptive_solve(state, pack, prob):
    """solve_fast with m_use from select_m when the config chooses K from an
    accuracy target (c3: AdaptivePolicy(epsilon=1e-3), adaptive.py:133-185)."""
    import paper_1607_04174_b200 as swb
    eps = state["params"].get("epsilon")
    if eps is None:
        return swb.solve_fast(pack, pack.laplacian, prob)
    m_use, _ = swb.select_m(pack, prob, swb.AdaptivePolicy(epsilon=eps))
    return swb.solve_fast(pack, pack.laplacian, prob, m_use=m_use)


def _round_prob(state, i):
    """c3's interaction rounds: step i solves with the seeds of rounds
    0..(i mod rounds) (100 more per label each round); else the fixed problem."""
    probs = state.get("round_probs")
    return probs[i % len(probs)] if probs else state["prob"]


def _fused(state) -> bool:
    """update_and_solve (the solve's reconstruction folded into the rotation)
    for the gamma = 0 configs with a fixed K; SWB_FUSED=0 times the two
    separate calls (update_basis, solve_fast) instead."""
    return (os.environ.get("SWB_FUSED", "1") != "0" and state.get("method") != "rayleigh"
            and state["prob"] is not None)


def _next_pack_and_solve(state, beta, i, prob):
    """_next_pack + solve_fast as one update_and_solve call (ping-pong V').

    c3 (K from an accuracy target, interaction rounds): every round updates
    the PRECOMPUTED pack to beta1 -- the reference's flow, nearest_pack(packs,
    beta) then the online update (cli.py:140-150) -- into one reused V'
    buffer.  Chaining first-order updates of updates (as the other configs'
    ping-pong does) accumulates the O(|dL|^2) loss of orthogonality step after
    step; after ~80 beta flips the seed rows of V' become ill-conditioned and
    select_m's seed fits leave the bidiagonal fast path (c3 step 11.7 -> 29
    ms, tools/step_drift.py), a state no reference user reaches."""
    import paper_1607_04174_b200 as swb
    eps = state["params"].get("epsilon")
    policy = swb.AdaptivePolicy(epsilon=eps) if eps is not None else None
    if policy is not None:
        base = state.setdefault("base", state["pack"])
        pack, field = swb.update_and_solve(base, state["image"], prob, state["params"]["beta1"],
                                           out=state.get("spare"), policy=policy)
        state["spare"] = pack.V
        state["pack"] = pack
        return field
    spare = state.pop("spare", None)
    old = state["pack"]
    cut = state.get("cut") if i % 2 == 0 else None
    pack, field = swb.update_and_solve(old, state["image"], prob, beta, cut_edges=cut, out=spare, policy=policy)
    state["spare"] = old.V
    state["pack"] = pack
    return field


def _registration_fused(state, beta, i, fixed, moving):
    """c5 through update_and_solve: the similarity priors first (they do not
    depend on the basis), then the update and the gamma > 0 solve with the
    reconstruction in the rotation, then the expected displacement."""
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import registration as R
    p = state["params"]
    pri = R.similarity_priors(fixed, moving, state["grid"], p["patch_radius"])
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(state["n"], [], []),
                            priors=pri.values_dev, gamma=p["gamma"])
    field = _next_pack_and_solve(state, beta, i, prob)
    field.displacement_dev = R.expected_displacement_device(field, state["grid"])
    return field


def gpu_step(state, i):
    p = state["params"]
    beta = p["beta1"] if i % 2 == 0 else p["beta0"]
    if state["prob"] is None and os.environ.get("SWB_FUSED", "1") != "0":
        return _registration_fused(state, beta, i, state["image"], state["moving"])
    if _fused(state):
        return _next_pack_and_solve(state, beta, i, _round_prob(state, i))
    pack = _next_pack(state, beta, i)
    if state["prob"] is None:
        return registration_solve(state, pack, state["image"], state["moving"])
    return _adaptive_solve(state, pack, _round_prob(state, i))


def e2e_step(state, i, host_labels):
    """Public API with host buffers: host seeds in (H2D inside solve_fast),
    host label map out (D2H into pinned memory) every step."""
    import paper_1607_04174_b200 as swb
    p = state["params"]
    beta = p["beta1"] if i % 2 == 0 else p["beta0"]
    if state["prob"] is None:
        # host fixed / moving images in (fresh Image objects: H2D every
        # step), host label map + displacement field out
        fixed = swb.Image(state["w"].dims, state["w"].intensities)
        moving = swb.Image(state["w"].dims, p["moving"])
        if os.environ.get("SWB_FUSED", "1") != "0":
            field = _registration_fused(state, beta, i, fixed, moving)
        else:
            pack = _next_pack(state, beta, i)
            field = registration_solve(state, pack, fixed, moving)
        host_labels.copy_(field.labels_dev, non_blocking=True)
        state["host_disp"].copy_(field.displacement_dev, non_blocking=True)
        return field
    seeds = _round_prob(state, i).seeds
    prob = swb.LabelProblem(num_labels=p["labels"],
                            seeds=swb.SeedPartition(state["n"], seeds.seed_indices.copy(), seeds.seed_labels.copy()))
    if _fused(state):
        field = _next_pack_and_solve(state, beta, i, prob)
    else:
        pack = _next_pack(state, beta, i)
        field = _adaptive_solve(state, pack, prob)
    host_labels.copy_(field.labels_dev, non_blocking=True)
    return field


def _ncu_traffic(kernel: str, cfg, dims, m):
    """DRAM bytes per launch of `kernel` from the committed ncu capture of the
    same workload (profiles/r2c_c4_kernel_metrics.json, tools/prof_r2c.sh), else None."""
    f = ROOT / "profiles" / "r2c_c4_kernel_metrics.json"
    if cfg != "c4" or dims is not None or m != 400 or not f.exists():
        return None
    try:
        return json.loads(f.read_text())["kernels"][kernel]["traffic_bytes"]
    except (KeyError, ValueError):
        return None


def fp64_probe(lib):
    """Live FP64 tensor-core peak: back-to-back DMMA.8x8x4 on every SM
    (swb_fp64_peak_probe), best of 5 after one warm-up, in TFLOP/s."""
    import torch

    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import stream_handle
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    flops = _lib.c_dbl()
    best = 0.0
    for it in range(6):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        _lib.check(lib.swb_fp64_peak_probe(20000, _lib.c_vp(sink.data_ptr()), _lib.C.byref(flops),
                                           stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        if it:
            best = max(best, flops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def int8_probe(lib, fn="swb_int8_peak_probe", iters=4000):
    """Live INT8 tensor-core peak: back-to-back tcgen05.mma.kind::i8
    (M 128, N 256, K 32) on every SM (swb_int8_peak_probe), best of 5 after
    one warm-up, in TOP/s.  fn="swb_int8_scheme_probe": the rotation GEMM's
    own MMA sequence (10 MMAs of N 64..256 per K chunk into seven group
    accumulators) -- the scheme's ceiling."""
    import torch

    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import stream_handle
    ops = _lib.C.c_double()
    best = 0.0
    for it in range(6):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        _lib.check(getattr(lib, fn)(iters, _lib.C.byref(ops), stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        if it:
            best = max(best, ops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def int8_sustained_probe(lib, seconds=1.5, pattern=0):
    """INT8 tensor-core rate with pseudo-random operands, held for ~seconds
    so the board reaches its power cap (the regime of the rotation GEMM inside
    the step): mean over the second half of back-to-back launches, TOP/s."""
    import torch

    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import stream_handle
    ops = _lib.C.c_double()
    iters = 40000 if pattern == 0 else 6000
    rates = []
    t_end = time.perf_counter() + seconds
    seed = 1
    while time.perf_counter() < t_end or len(rates) < 8:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        _lib.check(lib.swb_int8_probe_ex(pattern, iters, seed, _lib.C.byref(ops), stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        rates.append(ops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        seed += 1
    tail = rates[len(rates) // 2:]
    return float(np.mean(tail))


def measured_peaks() -> dict:
    mp = ROOT / "MEASURED_PEAKS.json"
    return json.loads(mp.read_text()) if mp.exists() else {}


def int8_denominator(peaks: dict, live_sustained: float | None):
    """INT8 roofline denominator: dense INT8 = 2 x dense bf16 on B200, and the
    rotation runs inside a long power-capped step, so 2 x the measured
    sustained cuBLAS bf16 rate (MEASURED_PEAKS.json); without that file, the
    live random-operand sustained probe."""
    if peaks.get("bf16_tflops_sustained"):
        return (2.0 * float(peaks["bf16_tflops_sustained"]),
                "of measured: 2 x MEASURED_PEAKS.json bf16_tflops_sustained (dense INT8 = 2 x dense bf16 on B200; "
                "sustained: the GEMM runs inside a long power-capped step)")
    return live_sustained, "live random-operand INT8 probe held ~1.5 s in this run (MEASURED_PEAKS.json absent)"


# the rotation's digit scheme (csrc/ozaki.cu): 7 digits per operand, the 28
# digit products with i + j <= 6, each an INT8 GEMM of the rotation's shape
OZ_PAIRS = 28


def run_sharded(args):
    """N > 1 ranks (torchrun): the c4 volume split into z-slabs, one per GPU
    (strong scaling).  Step = sharded first-order update (halo exchange +
    one all-reduce) + sharded RW solve (one all-reduce)."""
    import torch
    import torch.distributed as dist

    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200 import workloads as W
    from paper_1607_04174_b200.device import LatticeSpec
    from paper_1607_04174_b200.sharded import (CudaBackend, DistComm, Shard, SlabPlan, sharded_init_vtg,
                                                sharded_solve, sharded_update, sharded_update_and_solve)

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # stdout carries only rank 0's JSON line: NCCL writes its banner / logs
    # to file descriptor 1, so fd 1 points at stderr from here on and the
    # line goes to a duplicate of the original stdout
    json_out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
    m = args.m or W.CONFIGS[cfg]["m"]
    lib = _lib.load()
    w = W.make_image(cfg, dims)
    p = w.params
    n = int(np.prod(w.dims))
    lattice = LatticeSpec.make(w.dims, p["connectivity"], p["weight_mode"])
    plan = SlabPlan.make(w.dims, world, rank)
    # SWB_COMM=c: the collectives through the library's own NCCL entry points
    # (swb_comm_*, the C-host path) instead of torch.distributed
    if os.environ.get("SWB_COMM", "") == "c":
        from paper_1607_04174_b200.sharded import CComm
        comm = CComm(rank, world)
    else:
        comm = DistComm()
    be = CudaBackend()
    V = W.orthonormal_basis_slab(plan, m, W.CFG_INDEX[cfg] * 1000 + 17, comm)
    lam = torch.from_numpy(W.synthetic_lambda(cfg, m)).cuda()
    img = torch.from_numpy(np.array(w.intensities)).cuda()
    sh = Shard(plan, V, m, lam, lattice, img, be.graph(img, lattice, p["beta0"], plan=plan), p["beta0"])
    sharded_init_vtg([sh], comm, be)
    seeds, labs = W.seeds_for(w)

    fused = os.environ.get("SWB_FUSED", "1") != "0"

    def step(i):
        beta = p["beta1"] if i % 2 == 0 else p["beta0"]
        if fused:   # as the N = 1 step: the reconstruction rides in the rotation
            (labels, _, _, rc), = sharded_update_and_solve([sh], comm, be, beta, seeds, labs, p["labels"])
            return labels, rc
        sharded_update([sh], comm, be, beta)
        (labels, _, _, rc), = sharded_solve([sh], comm, be, seeds, labs, p["labels"])
        return labels, rc

    fp64_peak = fp64_probe(lib)
    int8_den, int8_den_src = int8_denominator(measured_peaks(), None)
    if int8_den is None:
        int8_den, int8_den_src = int8_denominator({}, int8_sustained_probe(lib))
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    from paper_1607_04174_b200 import api
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first()
    l0 = lib.swb_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(args.steps):
        labels, rc = step(args.warmup + i)
    e1.record()
    dist.barrier()
    torch.cuda.synchronize()
    launches = lib.swb_launch_count() - l0
    clk = clocks.stop()
    # phase breakdown from a second, untimed pass with events at the phase boundaries
    api.TIMER = api.PhaseTimer()
    for i in range(args.steps):
        labels, rc = step(args.warmup + i)
    torch.cuda.synchronize()
    phases = {k: float(np.mean(v)) for k, v in api.TIMER.durations().items()}
    api.TIMER = None
    ms_t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    # e2e: host seeds in, host labels out (each rank its slab) every step
    host = torch.empty(plan.own_end - plan.own_begin, dtype=torch.int32, pin_memory=True)
    dist.barrier()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(True), torch.cuda.Event(True)
    a0.record()
    for i in range(args.steps):
        labels, rc = step(args.warmup + args.steps + i)
        host.copy_(labels, non_blocking=True)
    a1.record()
    dist.barrier()
    torch.cuda.synchronize()
    et = torch.tensor([a0.elapsed_time(a1) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    ems = float(et.item())
    if rank == 0:
        line = {"metric": METRIC, "value": n * m / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{cfg}: {'x'.join(map(str, w.dims))} volume, K={m}, sharded first-order "
                                       f"update + {p['labels']}-label RW solve, S={len(seeds)}",
                           "N": n, "K": m, "parallelism": f"z-slab x{world} (halo Send/Recv + all-reduce, NCCL)",
                           "l2": "inputs larger than L2"},
                "e2e": {"value": n * m / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(len(seeds) * 12),
                        "d2h_bytes_per_step": int(n * 4 // world), "ms_per_step": ems},
                "gpu_launches": int(launches), "clocks": clk, "phases_ms": phases}
        rot_ms = phases.get("rotate")
        if rot_ms:
            rows = plan.own_end - plan.own_begin
            if m <= 512 and not os.environ.get("SWB_ROTATION", "").startswith("d"):
                ach = OZ_PAIRS * 2.0 * rows * m * m / (rot_ms * 1e-3) / 1e12
                line["roofline"] = {"bound": "tensor", "kernel": "rotation V*C on INT8 tcgen05 (digit split + "
                                    "GEMM), per GPU (rank 0 slab)", "achieved": ach, "peak": int8_den,
                                    "unit": "TOP/s (int8)", "frac": ach / int8_den,
                                    "peak_source": int8_den_src,
                                    "traffic": None, "algorithmic_bytes": 16.0 * rows * m}
            else:
                ach = 2.0 * rows * m * m / (rot_ms * 1e-3) / 1e12
                line["roofline"] = {"bound": "tensor", "kernel": "rotation V*C (DMMA NN GEMM), per GPU (rank 0 slab)",
                                    "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach / fp64_peak,
                                    "peak_source": "live DMMA.8x8x4 probe (swb_fp64_peak_probe) in this run",
                                    "traffic": None, "algorithmic_bytes": 16.0 * rows * m}
        print(json.dumps(line), file=json_out, flush=True)
    dist.destroy_process_group()


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import _lib, api
    from paper_1607_04174_b200 import workloads as W
    from paper_1607_04174_b200.device import stream_handle

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
    m = args.m or W.CONFIGS[cfg]["m"]
    lib = _lib.load()

    state = setup_gpu(cfg, dims, m, rank)
    state["method"] = args.method
    n = state["n"]
    if args.profile_steps:
        for i in range(args.profile_steps):
            gpu_step(state, i)
        torch.cuda.synchronize()
        return

    fp64_peak = fp64_probe(lib)
    int8_peak = int8_probe(lib)                   # zero operands, short: the burst figure
    scheme_peak = int8_probe(lib, "swb_int8_scheme_probe", 600)
    int8_sust = int8_sustained_probe(lib)         # random operands, held ~1.5 s: power-capped

    for i in range(args.warmup):
        gpu_step(state, i)
    torch.cuda.synchronize()
    if args.steps is None:
        # default K: 6 at c4 (a ~0.25 s step); smaller configs time enough
        # steps for ~1.5 s so the nvidia-smi sampler sees the loaded clock
        t0 = time.perf_counter()
        for i in range(2):
            gpu_step(state, args.warmup + i)
        torch.cuda.synchronize()
        per = (time.perf_counter() - t0) / 2
        args.steps = int(min(2000, max(6, round(1.5 / max(per, 1e-6)))))

    def barrier():
        if world > 1:
            dist.barrier()

    captured = None
    if args.graph:
        # two chained steps per graph (beta1 then back to beta0: the V' buffers
        # ping-pong back to where they started); the last pack's eigenvalues
        # and V'^T g are copied into the first pack's tensors so that every
        # replay continues the chain (swb.CapturedStep)
        if not _fused(state) or state["params"].get("epsilon") is not None:
            raise SystemExit("--graph: configs whose step is one update_and_solve at a fixed K (c1, c2, c4)")
        from paper_1607_04174_b200.capture import CapturedStep

        def two_steps():
            x = state["pack"]
            x.ensure_vtg()
            f0 = gpu_step(state, 0)
            f1 = gpu_step(state, 1)
            z = state["pack"]
            x.values_dev.copy_(z.values_dev)
            x.vtg.copy_(z.vtg)
            state["pack"], state["spare"] = x, state["spare"]
            return f0, f1

        captured = CapturedStep(two_steps)
        args.steps += args.steps % 2

    def run_steps(i0, k):
        if captured is None:
            for i in range(k):
                gpu_step(state, i0 + i)
        else:
            for _ in range(k // 2):
                captured.replay()

    # ---- device-resident timed region -------------------------------------
    # (no phase events inside it: the per-phase breakdown comes from a second,
    # untimed pass of the same K steps below)
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first()
    launches0 = lib.swb_launch_count()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    run_steps(args.warmup, args.steps)
    e1.record()
    barrier()
    torch.cuda.synchronize()
    launches = lib.swb_launch_count() - launches0
    if captured is not None:
        captured.check()
        # graph replays launch the captured kernels without passing the host
        # counter: count the library launches of one eager pair of steps
        c0 = lib.swb_launch_count()
        gpu_step(state, 0)
        gpu_step(state, 1)
        torch.cuda.synchronize()
        launches = (lib.swb_launch_count() - c0) * (args.steps // 2)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    # phase breakdown: the same steps again with CUDA events at every phase
    # boundary; per-step totals (a phase may repeat within a step: the
    # rotation's row chunks)
    api.TIMER = api.PhaseTimer()
    for i in range(args.steps):
        gpu_step(state, args.warmup + i)
    torch.cuda.synchronize()
    phases = {k: float(np.sum(v)) / args.steps for k, v in api.TIMER.durations().items()}
    api.TIMER = None
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = world * n * m / (ms * 1e-3)

    # ---- end-to-end through the public API with host buffers ---------------
    e2e = None
    if not args.no_e2e:
        host_labels = torch.empty(n, dtype=torch.int32, pin_memory=True)
        if state["prob"] is None:
            state["host_disp"] = torch.empty((n, 4), dtype=torch.float64, pin_memory=True)
        barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(True), torch.cuda.Event(True)
        a0.record()
        for i in range(args.steps):
            e2e_step(state, args.warmup + args.steps + i, host_labels)
        a1.record()
        barrier()
        torch.cuda.synchronize()
        ems = a0.elapsed_time(a1) / args.steps
        et = torch.tensor([ems], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        ems = float(et.item())
        s = state["seeds_n"]
        if state.get("round_probs"):   # mean seed count over the interaction rounds
            s = float(np.mean([pr.seeds.n_seeds for pr in state["round_probs"]]))
        if state["prob"] is None:
            h2d, d2h = 2 * n * 8, n * 4 + n * 4 * 8
        else:
            h2d, d2h = s * (8 + 4), n * 4 + 8
        e2e = {"value": world * n * m / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ------------------------------------
    rayleigh = args.method == "rayleigh"
    # the digit split of chunk i+1 overlaps the GEMM of chunk i: rotate_split
    # + rotate_join is its exposed part (the first chunk's split + any wait)
    rot_split_ms = (phases.get("rotate_split", 0.0) + phases.get("rotate_join", 0.0)) or None
    rot_gemm_ms = phases.get("rotate_gemm")
    rot_ms = sum(phases.get(k, 0.0) for k in ("rotate", "rotate_split", "rotate_gemm", "rotate_join")) or None
    rot_flops = 2.0 * n * m * m
    achieved = rot_flops / (rot_ms * 1e-3) / 1e12 if rot_ms else None
    peaks = measured_peaks()
    mp = ROOT / "MEASURED_PEAKS.json"
    hbm = float(peaks.get("hbm_gbs", 6650.0))   # fallback: B200_PROFILING.md
    proj_ms = phases.get("project")
    st_ms = phases.get("stencil")
    rc_ms = phases.get("solve_reconstruct")
    upd_ms = sum(v for k, v in phases.items() if not k.startswith("solve") and k not in ("priors", "displacement"))
    solve_ms = sum(v for k, v in phases.items() if k.startswith("solve") or k in ("priors", "displacement"))
    oz_tops = OZ_PAIRS * rot_flops / (rot_gemm_ms * 1e-3) / 1e12 if rot_gemm_ms else None
    kp = (m + 31) // 32 * 32
    split_bytes = 8.0 * n * m + 7.0 * n * kp + 8.0 * n
    kernels = {
        "rotation": {"ms": rot_ms, "fp64_equiv_tflops": achieved,
                     "note": "V*C: FP64 via INT8 tcgen05 digit products (split + GEMM); "
                             "SWB_ROTATION=dmma runs the DMMA GEMM instead"},
        "rotation_int8_gemm": {"ms": rot_gemm_ms, "int8_tops": oz_tops},
        "rotation_digit_split": {"ms_exposed": rot_split_ms, "bytes": split_bytes,
                                 "note": "chunk i+1 split on a side stream during GEMM i; ms = exposed part"},
        "projection_dmma": {"ms": proj_ms, "tflops": (n * m * (m + 1)) / (proj_ms * 1e-3) / 1e12 if proj_ms else None},
        "stencil_delta": {"ms": st_ms, "gbs": (16.0 * n * m + 72.0 * n) / (st_ms * 1e-3) / 1e9 if st_ms else None},
        "reconstruct_argmax": {"ms": rc_ms, "gbs": (8.0 * n * m + 20.0 * n) / (rc_ms * 1e-3) / 1e9 if rc_ms else None},
    }
    if not rot_gemm_ms and rot_ms:   # DMMA rotation (m > 512 or SWB_ROTATION=dmma)
        kernels["rotation"]["frac_fp64"] = achieved / fp64_peak
    L = state["params"]["labels"]
    fz_ms = phases.get("solve_finalize")
    if fz_ms and not rc_ms:   # update_and_solve: V' coeff came out of the rotation's padding columns
        del kernels["reconstruct_argmax"]
        kernels["finalize_argmax"] = {
            "ms": fz_ms, "gbs": (8.0 * L + 20.0) * n / (fz_ms * 1e-3) / 1e9,
            "note": "update_and_solve: the reconstruction V' coeff = V (C coeff) rides in the rotation GEMM's "
                    "padding columns; this pass reads the N x L products + d_sqrt, writes labels / top-2"}
        kernels["finalize_argmax"]["frac_hbm"] = kernels["finalize_argmax"]["gbs"] / hbm
    if L > 8 and rc_ms:   # many labels: V (coeff) on the DMMA GEMM, then the finalize / argmax pass
        kernels["reconstruct_argmax"] = {"ms": rc_ms, "tflops": 2.0 * n * m * L / (rc_ms * 1e-3) / 1e12,
                                         "note": "NN GEMM N x K x L + finalize/argmax pass"}
    for k in ("projection_dmma", "reconstruct_argmax"):
        if k in kernels and kernels[k].get("tflops"):
            kernels[k]["frac_fp64"] = kernels[k]["tflops"] / fp64_peak
    for k in ("stencil_delta", "reconstruct_argmax"):
        if k in kernels and kernels[k].get("gbs"):
            kernels[k]["frac_hbm"] = kernels[k]["gbs"] / hbm
    if rayleigh:   # the reference's refresh: one read-only stencil pass over V (HBM)
        sr_ms = phases.get("stencil_rayleigh")
        kernels = {k: v for k, v in kernels.items()
                   if not k.startswith("rotation") and k not in ("projection_dmma", "stencil_delta")}
        kernels["stencil_rayleigh"] = {"ms": sr_ms, "gbs": (8.0 * n * m + 48.0 * n) / (sr_ms * 1e-3) / 1e9
                                       if sr_ms else None}
        if sr_ms:
            kernels["stencil_rayleigh"]["frac_hbm"] = kernels["stencil_rayleigh"]["gbs"] / hbm

    # INT8 denominator (int8_denominator); the zero-operand burst probe and
    # the live random-operand sustained probe are reported beside it
    int8_den, int8_den_src = int8_denominator(peaks, int8_sust)
    # the dominant kernel by time: the INT8 rotation GEMM or the DMMA projection
    # (the INT8 rotation's own roofline is kept under kernels either way)
    rot_roof = None
    if rot_gemm_ms:
        rot_roof = {"bound": "tensor", "kernel": "rotation V*C: INT8 tcgen05 digit-product GEMM (oz_gemm_kernel)",
                    "achieved": oz_tops, "peak": int8_den, "unit": "TOP/s (int8)",
                    "frac": oz_tops / int8_den if oz_tops else None,
                    "peak_source": int8_den_src,
                    "peak_burst_zero_operands": int8_peak,
                    "peak_burst_source": "live tcgen05.mma.kind::i8 M128xN256 probe on zero-filled shared memory, "
                                         "2 ms launches (swb_int8_peak_probe): burst clock, no operand switching",
                    "peak_live_random_sustained": int8_sust,
                    "frac_of_live_random_sustained": oz_tops / int8_sust if oz_tops and int8_sust else None,
                    "peak_live_random_sustained_source": "the same MMA stream on pseudo-random operand bytes, "
                                                         "back-to-back for ~1.5 s (swb_int8_probe_ex)",
                    "algorithmic": f"{OZ_PAIRS} digit products x 2*N*K*K ops",
                    "traffic": _ncu_traffic("rotation_int8_gemm", cfg, dims, m),
                    "algorithmic_bytes": 16.0 * n * m,
                    # the scheme's own ceiling: the GEMM's MMA sequence alone
                    # (10 MMAs of N = 64..256 per K chunk into the seven
                    # resident int32 group accumulators), swb_int8_scheme_probe
                    "scheme_peak": scheme_peak,
                    "frac_of_scheme_peak": oz_tops / scheme_peak if oz_tops and scheme_peak else None,
                    "scheme_peak_source": "live probe of the GEMM's MMA sequence alone (M128 K32 SS, the 28 digit "
                                          "products of a K chunk as 10 MMAs of N = 64..256 into 7 TMEM group "
                                          "accumulators; swb_int8_scheme_probe) in this run"}
        kernels["rotation_int8_gemm"].update(
            {k: rot_roof[k] for k in ("frac", "peak", "frac_of_live_random_sustained", "scheme_peak",
                                      "frac_of_scheme_peak", "traffic")})
    if rot_roof and (not proj_ms or rot_gemm_ms >= proj_ms):
        roofline = rot_roof
    else:
        pj = kernels["projection_dmma"]["tflops"] if proj_ms else None
        roofline = {"bound": "tensor", "kernel": "projection V^T(dL V) (DMMA TN GEMM, symmetric)",
                    "achieved": pj, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": pj / fp64_peak if pj else None,
                    "peak_source": "live DMMA.8x8x4 probe (swb_fp64_peak_probe) in this run; MEASURED_PEAKS.json "
                                   "has no FP64 entry",
                    "traffic": _ncu_traffic("projection_tn_sym", cfg, dims, m),
                    "algorithmic_bytes": 16.0 * n * m}
        if not rot_gemm_ms and rot_ms and (not proj_ms or rot_ms >= proj_ms):
            roofline = {"bound": "tensor", "kernel": "rotation V*C (DMMA NN GEMM)", "achieved": achieved,
                        "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak if achieved else None,
                        "peak_source": "live DMMA.8x8x4 probe (swb_fp64_peak_probe) in this run",
                        "traffic": _ncu_traffic("rotation_nn", cfg, dims, m), "algorithmic_bytes": 16.0 * n * m}

    cpu = None
    if not args.no_cpu:
        try:
            cpu = cpu_baseline(cfg, dims, m)
        except Exception as exc:  # noqa: BLE001 - reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}

    dims_full = tuple(state["w"].dims)
    s = state["seeds_n"]
    rp = state.get("round_probs")
    solve_desc = (f"{state['params']['labels']}-label RW solve, S={s}" if not rp else
                  f"{state['params']['labels']}-label RW solve with K from select_m(epsilon="
                  f"{state['params']['epsilon']}), {len(rp)} interaction rounds cycled (S = "
                  f"{rp[0].seeds.n_seeds}..{rp[-1].seeds.n_seeds})")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if world > 1 else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg}: {'x'.join(map(str, dims_full))} volume, K={m}, "
                               f"{'refresh (reference, eigenvalue-only)' if rayleigh else 'first-order'} " + (
                                   f"topology update (cut <-> restore the edges crossing a "
                                   f"{state['params']['cut_block']}x{state['params']['cut_block']} block boundary, "
                                   f"beta {state['params']['beta0']}) + " if state.get("cut") is not None else
                                   (f"beta update {state['params']['beta0']}->{state['params']['beta1']} of the "
                                    f"precomputed pack every round + " if rp else
                                    f"beta update {state['params']['beta0']}<->{state['params']['beta1']} + ")) + (
                                   solve_desc if cfg != "c5" else
                                   f"similarity priors (grid {state['params']['grid']}, patch radius "
                                   f"{state['params']['patch_radius']}) + {state['params']['labels']}-label "
                                   f"gamma={state['params']['gamma']} RW solve + expected displacement"),
                   "N": n, "K": m, "labels": state["params"]["labels"], "seeds": int(s),
                   "parallelism": "replicas" if world > 1 else "single",
                   "cuda_graph": bool(getattr(args, "graph", False)),
                   "l2": "inputs larger than L2 (V = %.1f GB)" % (n * m * 8 / 1e9)},
        "roofline": ({"bound": "hbm", "kernel": "refresh Rayleigh stencil pass (read V once)",
                      "achieved": kernels["stencil_rayleigh"]["gbs"], "peak": hbm, "unit": "GB/s",
                      "frac": kernels["stencil_rayleigh"].get("frac_hbm"), "traffic": None,
                      "algorithmic_bytes": 8.0 * n * m + 48.0 * n} if rayleigh else None) or
                    roofline,
        "kernels": kernels,
        "peaks": {"fp64_tflops": fp64_peak, "fp64_source": "of measured: live DMMA probe in this run",
                  "int8_tops": int8_den, "int8_source": int8_den_src,
                  "int8_tops_burst_zero_operands": int8_peak, "int8_tops_live_random_sustained": int8_sust,
                  "hbm_gbs": hbm, "hbm_source": "of measured: MEASURED_PEAKS.json hbm_gbs" if mp.exists()
                  else "of fallback: B200_PROFILING.md"},
        "update": {"ms": upd_ms, "value": n * m / (upd_ms * 1e-3) if upd_ms else None, "unit": UNIT},
        "solve": {"ms": solve_ms, "value": n / (solve_ms * 1e-3) if solve_ms else None, "unit": "voxels/s"},
        "phases_ms": phases,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.steps is None and (args.impl == "reference" or int(os.environ.get("WORLD_SIZE", "1")) > 1
                               or args.sharded):
        args.steps = 6
    if args.impl == "reference":
        run_reference(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.sharded:
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"), ("MASTER_ADDR", "127.0.0.1"),
                     ("MASTER_PORT", "29533")):
            os.environ.setdefault(k, v)
        run_sharded(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
