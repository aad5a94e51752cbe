"""Randomised parity sweep of the public filter against the numpy oracle
(tests/_fuzz_cases.py): python tools/gpu/fuzz.py [cases] [seed]; SBF_FUZZ_VARIANT=2 runs
CUDA-tensor inputs through the warp-specialised K3 sweep.  Exit code 1 if any case fails."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from _fuzz_cases import run_cases  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
var = os.environ.get("SBF_FUZZ_VARIANT")
fails = run_cases(n, seed, variant=int(var) if var else None, log=lambda m: print(m, flush=True))
print(f"{n} cases, {len(fails)} failing")
sys.exit(1 if fails else 0)
