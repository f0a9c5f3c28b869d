"""swb.install on a caller tree with the reference's binding pattern, on the
GPU: the caller's from-imported solve_fast / select_m / hard_labels /
refresh_from_set run the B200 path, and a host pack passed to repeated calls
is uploaded to the device once.

The GPU box has no reference tree, so the caller package here is a small
stand-in written for this test: modules that define the hot-path names and a
``cli`` module that from-imports them and calls them in the order of the
reference's ``_cmd_segment`` (cli.py:126-163).  tests/test_dropin_cpu.py runs
``install`` on the real reference package (binding checks)."""

import importlib
import sys
import textwrap

import numpy as np
import pytest

from oracle import rw_oracle as O

pytestmark = pytest.mark.gpu

FILES = {
    "__init__.py": """
        from .fastrw import solve_fast
        from .adaptive import select_m
        from .images import hard_labels
        from .refresh import refresh, refresh_from_set, nearest_pack
    """,
    "fastrw.py": """
        def solve_fast(pack, lap, prob, m_use=None, streaming_block=None):
            raise RuntimeError("host path called")
    """,
    "adaptive.py": """
        def select_m(pack, prob, policy=None):
            raise RuntimeError("host path called")
    """,
    "images.py": """
        def hard_labels(field):
            raise RuntimeError("host path called")
    """,
    "refresh.py": """
        def refresh(pack, image, new_beta):
            raise RuntimeError("host path called")
        def nearest_pack(packs, new_beta):
            raise RuntimeError("host path called")
        def refresh_from_set(packs, image, new_beta):
            return refresh(nearest_pack(packs, new_beta), image, new_beta)
    """,
    "cli.py": """
        from .adaptive import select_m
        from .fastrw import solve_fast
        from .images import hard_labels
        from .refresh import refresh_from_set

        def segment(packs, image, prob, policy, beta_online=None, lap=None, adaptive=False):
            if beta_online is not None:
                pack = refresh_from_set(packs, image, beta_online)
                lap = pack.laplacian
            else:
                pack = packs.packs[0]
            m_use = select_m(pack, prob, policy)[0] if adaptive else pack.m
            field = solve_fast(pack, lap, prob, m_use=m_use)
            return hard_labels(field), field, m_use
    """,
}


@pytest.fixture()
def fake_ref(tmp_path):
    root = tmp_path / "swb_fake_ref"
    root.mkdir()
    for name, body in FILES.items():
        (root / name).write_text(textwrap.dedent(body))
    sys.path.insert(0, str(tmp_path))
    try:
        yield importlib.import_module("swb_fake_ref")
    finally:
        sys.path.remove(str(tmp_path))
        for k in [k for k in sys.modules if k.startswith("swb_fake_ref")]:
            del sys.modules[k]


def _case():
    dims, conn, mode, m = (40, 36), 4, "abs", 40
    rng = np.random.default_rng(3)
    n = dims[0] * dims[1]
    xs, ys = np.meshgrid(np.arange(dims[0]), np.arange(dims[1]), indexing="ij")
    img = np.where((xs - 20) ** 2 + (ys - 18) ** 2 <= 100, 0.7, 0.3).reshape(-1, order="F")
    img = np.clip(img + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 15.0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    seeds = np.sort(rng.choice(n, 24, replace=False))
    labs = (img[seeds] > 0.5).astype(np.int64)
    return dims, img, lap0, vecs[:, :m], vals[:m], seeds, labs


def test_installed_callers_run_on_gpu_with_one_upload(cuda_ok, fake_ref):
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import api
    from paper_1607_04174_b200._lib import load
    dims, img, lap0, V, lam, seeds, labs = _case()
    n = img.size
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=15.0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    packs = swb.PackSet((pack,))
    prob = swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(n, seeds, labs))
    cli = importlib.import_module("swb_fake_ref.cli")
    with swb.install(fake_ref) as inst:
        assert ("swb_fake_ref.cli", "solve_fast") in inst.replaced
        assert ("swb_fake_ref.cli", "refresh_from_set") in inst.replaced
        up0 = api.UPLOADS[0]
        lib = load()
        launches0 = lib.swb_launch_count()
        # fixed beta, reference Laplacian (cli.py:149-150), three solves on one host pack
        for _ in range(3):
            lab, field, m_use = cli.segment(packs, image, prob, swb.AdaptivePolicy(), lap=lap0)
        assert api.UPLOADS[0] - up0 == 1, "host pack uploaded more than once"
        assert lib.swb_launch_count() > launches0
        u_ref = O.solve_fast(V, lam, lap0.d_sqrt, lap0.matrix, seeds, labs, 2)
        np.testing.assert_allclose(field.values, u_ref, rtol=0, atol=1e-10)
        gap = O.top2_gap(u_ref)
        assert not ((lab.labels != O.hard_labels(u_ref)) & (gap >= 1e-9)).any()
        # beta-online through the caller's refresh_from_set + adaptive select_m
        lab2, field2, m2 = cli.segment(packs, image, prob, swb.AdaptivePolicy(epsilon=0.5), beta_online=20.0,
                                       adaptive=True)
        assert api.UPLOADS[0] - up0 == 1
        lap1 = O.build_laplacian(img, dims, 20.0, "abs", 4)
        lam_r, order = O.refresh(V, lap1)
        m_o, _ = O.select_m(V[:, order], lap1.d_sqrt, seeds, labs, 2, epsilon=0.5)
        assert m2 == m_o
        u2 = O.solve_fast(V[:, order], lam_r, lap1.d_sqrt, lap1.matrix, seeds, labs, 2, m_use=m_o)
        np.testing.assert_allclose(field2.values, u2, rtol=0, atol=1e-10)
    # uninstalled: the caller is back on its own functions
    with pytest.raises(RuntimeError, match="host path"):
        cli.segment(packs, image, prob, swb.AdaptivePolicy(), lap=lap0)
