"""The unmodified reference package's own callers on the B200 path, GPU.

`baseline/_ref` holds the reference package installed unmodified by pip
(`pip install --no-index --no-deps --target baseline/_ref <copy of
/root/reference/pkg>`); it travels to the GPU box with the
repo snapshot (git-ignored, not gpurun-ignored).  With it present this test
runs the reference CLI `segment` command (cli.py:126-163) and the service
`SessionStore` (service/sessions.py:61-157) twice on the same files: once
as shipped (its CPU numpy/scipy path) and once after `swb.install(specwalk)`
(the B200 kernels), and compares what the callers write / return.  Skipped
when `baseline/_ref` is absent (nothing here reads /root/reference)."""

import importlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def specwalk():
    if not (REF / "specwalk" / "__init__.py").exists():
        pytest.skip("baseline/_ref (the pip-installed reference) not present")
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    try:
        yield importlib.import_module("specwalk")
    finally:
        sys.path.remove(str(REF))


def _files(sw, tmp_path, dims=(40, 36), m=30, betas=(15.0, 30.0)):
    """Image (RAWJ), two packs (.rwpk, the reference writer) and seeds (JSON)."""
    rng = np.random.default_rng(11)
    n = int(np.prod(dims))
    xs, ys = np.meshgrid(np.arange(dims[0]), np.arange(dims[1]), indexing="ij")
    img = np.where((xs - 20) ** 2 + (ys - 17) ** 2 <= 110, 0.7, 0.3).reshape(-1, order="F")
    img = np.clip(img + rng.normal(0, 0.05, n), 0, 1).astype(np.float32).astype(np.float64)
    img_path = sw.images.save_image(sw.Image(dims=dims, intensities=img), tmp_path / "img")
    image = sw.load_image(img_path)
    packs = []
    for beta in betas:
        lap = sw.laplacian(sw.build_graph(image, beta), sw.LaplacianMode.NORMALIZED)
        lam, V = np.linalg.eigh(lap.matrix.toarray())
        pack = sw.SpectralPack(dims=image.dims, spacing=image.spacing, beta=beta,
                               eigen=sw.EigenBasis(np.asfortranarray(V[:, :m]), lam[:m]), d_sqrt=lap.d_sqrt,
                               provenance=sw.fastrw.PackProvenance(image_hash=image.content_hash()))
        path = tmp_path / f"p{beta:g}.rwpk"
        sw.save_pack(pack, path)
        packs.append(str(path))
    inside = np.flatnonzero(img > 0.5)
    outside = np.flatnonzero(img <= 0.5)
    seeds = [{"index": int(i), "label": 1} for i in rng.choice(inside, 12, replace=False)] + \
            [{"index": int(i), "label": 0} for i in rng.choice(outside, 12, replace=False)]
    seeds_path = tmp_path / "seeds.json"
    seeds_path.write_text(json.dumps(seeds))
    return str(img_path), packs, str(seeds_path)


def _segment(sw, args, prefix):
    rc = sw.cli.main(["segment", *args, "--out-prefix", str(prefix)])
    assert rc == 0
    lab = sw.images.load_labels(str(prefix) + "_labels")
    prob = sw.images.load_probabilities(str(prefix) + "_probs")
    return lab.labels, prob.values


@pytest.mark.parametrize("extra", [[], ["--beta-online", "20"], ["--beta-online", "24", "--adaptive",
                                                                  "--epsilon", "0.3"], ["--m-use", "12"]])
def test_reference_cli_segment_on_gpu_matches_reference(cuda_ok, specwalk, tmp_path, extra, capsys):
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import api
    from paper_1607_04174_b200._lib import load
    sw = specwalk
    importlib.import_module("specwalk.cli")
    img, packs, seeds = _files(sw, tmp_path)
    args = [img, *packs, seeds, *extra]
    lab_cpu, p_cpu = _segment(sw, args, tmp_path / "cpu")
    rep_cpu = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    lib = load()
    with swb.install(sw) as inst:
        assert ("specwalk.cli", "solve_fast") in inst.replaced
        l0, u0 = lib.swb_launch_count(), api.UPLOADS[0]
        lab_gpu, p_gpu = _segment(sw, args, tmp_path / "gpu")
        rep_gpu = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
        assert lib.swb_launch_count() > l0, "the CLI did not reach the B200 kernels"
        assert api.UPLOADS[0] - u0 <= 1
    assert rep_gpu["m_use"] == rep_cpu["m_use"] and rep_gpu["refreshed"] == rep_cpu["refreshed"]
    assert rep_gpu["base_beta"] == rep_cpu["base_beta"]
    # probabilities are written as f32 (images.py:269-271): equal to f32 rounding
    np.testing.assert_allclose(p_gpu, p_cpu, rtol=0, atol=2e-7)
    srt = np.sort(p_cpu, axis=1)
    tie = (srt[:, -1] - srt[:, -2]) < 1e-6
    assert not ((lab_gpu != lab_cpu) & ~tie).any()


def test_reference_session_store_on_gpu_matches_reference(cuda_ok, specwalk, tmp_path):
    """SessionStore.create / update_params (beta refresh, sessions.py:95-121)
    / solve (select_m + solve_fast + argmax, :123-157) on the B200 path."""
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200._lib import load
    sw = specwalk
    sessions = pytest.importorskip("specwalk.service.sessions")
    img, packs, seeds_path = _files(sw, tmp_path)
    raw = json.loads(Path(seeds_path).read_text())
    image = sw.load_image(img)
    seeds = sw.SeedPartition(image.n_voxels, [s["index"] for s in raw], [s["label"] for s in raw])

    def run():
        store = sessions.SessionStore()
        sess = store.create(img, packs, gamma=0.0, epsilon=0.3, beta=None)
        r1 = store.solve(sess, seeds, adaptive=True)
        store.update_params(sess, beta=22.0)
        r2 = store.solve(sess, seeds, adaptive=False, m_use=20)
        return r1, r2

    c1, c2 = run()
    lib = load()
    with swb.install(sw):
        l0 = lib.swb_launch_count()
        g1, g2 = run()
        assert lib.swb_launch_count() > l0
    for c, g in ((c1, g1), (c2, g2)):
        assert c.m_use == g.m_use and c.num_labels == g.num_labels
        assert np.mean(c.labels != g.labels) < 1e-3          # argmax off exact ties
        assert np.abs(c.max_prob.astype(int) - g.max_prob.astype(int)).max() <= 1
