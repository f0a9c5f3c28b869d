"""Route the reference package's own callers to this library.

The reference (``specwalk``) binds its hot-path functions into its callers
with ``from … import`` at import time:

  cli.py:17-23              select_m, solve_fast, hard_labels, refresh_from_set (+ load_pack)
  service/sessions.py:17-23 select_m, solve_fast, refresh_from_set (+ load_pack)
  registration.py:16-20     select_m, solve_fast
  bench.py:19-23            select_m, solve_fast, hard_labels
  __init__.py:3-28          the package-level names

so assigning ``specwalk.solve_fast = …`` reaches none of them.  ``install``
rebinds every module-level name that still *is* the reference function
(identity check, so unrelated same-named attributes are never touched) in
the package, its defining modules and every caller module, and returns an
``Installation`` whose ``uninstall()`` restores them.  After it,
``specwalk.cli._cmd_segment`` (cli.py:126-163), ``SessionStore.solve``
(service/sessions.py:123-157), ``SessionStore._apply_beta`` (:95-104) and
``register`` (registration.py:216-225) run the B200 path.

Host packs handed in by those callers are uploaded once per pack object
(``api._as_device`` caches the device copy), results come back as
``DeviceField`` objects exposing the ``ProbabilityField`` surface the callers
read (``values``, ``K``, ``dims``, ``clamped()``), and ``hard_labels`` returns
the reference ``LabelMap`` layout (``dims``, ``labels``).
"""

from __future__ import annotations

import importlib
import sys
from dataclasses import dataclass, field

# hot-path names -> (defining reference module, our function name)
HOT_PATH = {
    "solve_fast": ("fastrw", "solve_fast"),
    "select_m": ("adaptive", "select_m"),
    "hard_labels": ("images", "hard_labels"),
    "refresh": ("refresh", "refresh"),
    "refresh_from_set": ("refresh", "refresh_from_set"),
    "nearest_pack": ("refresh", "nearest_pack"),
}
# opt-in: .rwpk ingest (fastrw.py:264-325, native xxh64 + GPU transpose) and
# the GPU offline precompute (fastrw.py:200-221); load_pack then returns device
# packs, so save_pack must follow it
PACK_IO = {
    "load_pack": ("fastrw", "load_pack"),
    "save_pack": ("fastrw", "save_pack"),
}
PRECOMPUTE = {
    "precompute": ("fastrw", "precompute"),
}
# modules that bind the names at import time (the callers) and the defining ones
CALLERS = ("fastrw", "refresh", "adaptive", "images", "cli", "registration", "bench", "service.sessions",
           "service.app")


@dataclass
class Installation:
    package: str
    replaced: list = field(default_factory=list)      # (module name, attribute name)
    skipped: dict = field(default_factory=dict)       # module name -> import error text
    _saved: list = field(default_factory=list, repr=False)

    def uninstall(self) -> None:
        for mod, name, orig in reversed(self._saved):
            setattr(mod, name, orig)
        self._saved.clear()
        self.replaced.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()


def _ours(name: str):
    from . import api, packs
    pre = importlib.import_module(__package__ + ".precompute")   # the package attr is the function
    table = {"solve_fast": api.solve_fast, "select_m": api.select_m, "hard_labels": api.hard_labels,
             "refresh": api.refresh, "refresh_from_set": api.refresh_from_set, "nearest_pack": api.nearest_pack,
             "load_pack": packs.load_pack, "save_pack": packs.save_pack, "precompute": pre.precompute}
    return table[name]


def install(specwalk=None, *, pack_io: bool = False, precompute: bool = False) -> Installation:
    """Rebind the reference's hot path inside ``specwalk`` (module or name).

    Needs no GPU to install; the rebound functions need one when called
    (no CPU fallback: they raise ``BackendUnavailable`` without a device).
    """
    if specwalk is None or isinstance(specwalk, str):
        specwalk = importlib.import_module(specwalk or "specwalk")
    pkg = specwalk.__name__
    names = dict(HOT_PATH)
    if pack_io:
        names.update(PACK_IO)
    if precompute:
        names.update(PRECOMPUTE)
    inst = Installation(pkg)
    modules = {pkg: specwalk}
    for sub in CALLERS:
        full = f"{pkg}.{sub}"
        try:
            modules[full] = importlib.import_module(full)
        except Exception as exc:   # optional callers (e.g. the FastAPI app without fastapi)
            inst.skipped[full] = f"{type(exc).__name__}: {exc}"
    # any other already-imported submodule binds the names too
    for full, mod in list(sys.modules.items()):
        if full.startswith(pkg + ".") and mod is not None and full not in modules:
            modules[full] = mod
    originals = {}
    for name, (defmod, _) in names.items():
        mod = modules.get(f"{pkg}.{defmod}")
        if mod is not None and hasattr(mod, name):
            originals[name] = getattr(mod, name)
    for full, mod in modules.items():
        for name, orig in originals.items():
            if getattr(mod, name, None) is orig:
                inst._saved.append((mod, name, orig))
                setattr(mod, name, _ours(name))
                inst.replaced.append((full, name))
    return inst
