"""Run bench.py with every torch.empty pre-filled with NaN (debugging aid: a
kernel that lets padding reach a result then fails in the step's own checks).
python tools/nanfill_bench.py --config c5 --no-cpu"""
import runpy
import sys
from pathlib import Path

import torch

torch.use_deterministic_algorithms(True, warn_only=True)
torch.utils.deterministic.fill_uninitialized_memory = True
sys.argv = [str(Path(__file__).resolve().parent.parent / "bench.py")] + sys.argv[1:]
runpy.run_path(sys.argv[0], run_name="__main__")
