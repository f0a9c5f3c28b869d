"""Build a compile-time variant of the library for A/B timing:
python tools/build_variant.py OUT.so -DSWB_ST_PREF=3 ...  (then SWB_LIB=OUT.so python bench.py)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1607_04174_b200 import build_ext as B  # noqa: E402


def main():
    out = Path(sys.argv[1]).resolve()
    defs = sys.argv[2:]
    nvcc = B.nvcc_path()
    objdir = out.parent / (out.stem + "_obj")
    objdir.mkdir(parents=True, exist_ok=True)
    flags = B.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-prec-div=true", "-prec-sqrt=true",
                      "-I", str(ROOT / "include"), *defs]
    procs = []
    objs = []
    for src in B.SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        objs.append(str(obj))
        procs.append(subprocess.Popen([nvcc, *flags, "-c", str(B.CSRC / src), "-o", str(obj)]))
    if any(p.wait() for p in procs):
        raise SystemExit("compile failed")
    subprocess.run([nvcc, *B.ARCH, "-shared", "-cudart=static", "-o", str(out), *objs, "-ldl"], check=True)
    print(out)


if __name__ == "__main__":
    main()
