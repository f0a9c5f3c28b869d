"""CPU guard for GPU-only code paths: every name loaded in the package's
Python modules is defined somewhere in that module (import, def, class,
assignment, argument) or is a builtin.  Catches NameErrors in branches the
CPU suite cannot execute."""

import ast
import builtins
from pathlib import Path

import pytest

PKG = Path(__file__).resolve().parents[1] / "paper_1607_04174_b200"


def _undefined(src: str) -> set:
    tree = ast.parse(src)
    defined = set(dir(builtins)) | {"__file__", "__name__"}
    for node in ast.walk(tree):
        if isinstance(node, (ast.FunctionDef, ast.AsyncFunctionDef, ast.ClassDef)):
            defined.add(node.name)
        elif isinstance(node, ast.Import):
            defined.update((a.asname or a.name).split(".")[0] for a in node.names)
        elif isinstance(node, ast.ImportFrom):
            defined.update(a.asname or a.name for a in node.names)
        elif isinstance(node, ast.arg):
            defined.add(node.arg)
        elif isinstance(node, ast.ExceptHandler) and node.name:
            defined.add(node.name)
        targets = []
        if isinstance(node, ast.Assign):
            targets = node.targets
        elif isinstance(node, (ast.AnnAssign, ast.AugAssign, ast.NamedExpr)):
            targets = [node.target]
        elif isinstance(node, (ast.For, ast.comprehension)):
            targets = [node.target]
        elif isinstance(node, ast.With):
            targets = [it.optional_vars for it in node.items if it.optional_vars is not None]
        for t in targets:
            defined.update(n.id for n in ast.walk(t) if isinstance(n, ast.Name))
    used = {n.id for n in ast.walk(tree) if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Load)}
    return used - defined


@pytest.mark.parametrize("mod", sorted(p.name for p in PKG.glob("*.py")))
def test_no_undefined_names(mod):
    assert _undefined((PKG / mod).read_text()) == set()


def test_bench_no_undefined_names():
    assert _undefined((PKG.parent / "bench.py").read_text()) == set()
