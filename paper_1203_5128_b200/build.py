"""Build libsbf.so (sm_100a) in-tree with nvcc; no torch extension machinery.

    python -m paper_1203_5128_b200.build [--full|--min] [-j N]

Each specialised K3 instantiation (r, passes, precision mode) is its own
object so the build parallelises.  The instantiation list is written to
csrc/sbf_terms_list.inc, which the dispatcher includes.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsbf.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-Xptxas", "-warn-spills", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", INCLUDE, "-I", CSRC] + os.environ.get("SBF_NVCC_FLAGS", "").split()

SOURCES = ["sbf_api.cu", "sbf_plan.cu", "sbf_local_range.cu", "sbf_generic.cu", "sbf_pgm.cu",
           "sbf_direct.cu", "sbf_nlm.cu", "sbf_dual.cu", "sbf_smooth.cu", "sbf_stage.cu"]


def instantiations(kind: str):
    """(r, passes, mode) triples with a specialised K3 kernel."""
    # HDR (mode 1) has no specialised kernel yet: it runs the fp64 generic path
    if kind == "min":
        return [(2, 3, 0), (4, 3, 0), (5, 3, 0)]
    out = []
    for r in range(0, 13):
        out.append((r, 3, 0))
    for r in range(1, 13):
        out.append((r, 1, 0))
    return out


def split_instantiations(kind: str):
    """(r, passes) pairs with a split-sweep (SV/SH) instantiation."""
    if kind == "min":
        return [(5, 3)]
    # (single-pass boxes of radius 6..12 too: every fp32 radius >= 6 is then
    # served by the bit-reproducible split sweep)
    return [(r, 3) for r in range(5, 13)] + [(r, 1) for r in range(6, 13)]


def sweep_instantiations(kind: str):
    """(r, passes) pairs with a K3 sweep instantiation (four images per V
    thread: the 2r+3 register rings of 3 passes fit up to r = 5)."""
    if kind == "min":
        return [(2, 3), (4, 3), (5, 3)]
    return [(r, 3) for r in range(0, 6)] + [(r, 1) for r in range(1, 6)]


def _newer(target, deps):
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h", ".inc"))]
    hs.append(os.path.join(INCLUDE, "sbf.h"))
    return hs


def _compile(args):
    src, obj, defs = args
    deps = [src] + _headers()
    if _newer(obj, deps):
        return obj, 0, ""
    cmd = [NVCC] + ARCH + FLAGS + defs + ["-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    return obj, p.returncode, p.stdout + p.stderr


def build(kind: str = "full", jobs: int | None = None, verbose: bool = False,
          variant: str | None = None, defs: list[str] | None = None) -> str:
    """Compile and link.  `variant` + `defs` build an experimental copy
    (extra -D flags on every object) into _build_<variant>/libsbf_<variant>.so,
    loadable with SBF_LIB=...; the default library is untouched."""
    obj_dir, lib = OBJ, LIB
    defs = list(defs or [])
    if variant:
        obj_dir = OBJ + "_" + variant
        lib = os.path.join(HERE, f"libsbf_{variant}.so")
    os.makedirs(obj_dir, exist_ok=True)
    inst = instantiations(kind)
    inc = os.path.join(CSRC, "sbf_terms_list.inc")
    text = "".join(f"SBF_X({r}, {p}, {m})\n" for r, p, m in inst)
    if not os.path.exists(inc) or open(inc).read() != text:
        with open(inc, "w") as fh:
            fh.write(text)
    sinst = split_instantiations(kind)
    sinc = os.path.join(CSRC, "sbf_split_list.inc")
    stext = "".join(f"SBF_Y({r}, {p})\n" for r, p in sinst)
    if not os.path.exists(sinc) or open(sinc).read() != stext:
        with open(sinc, "w") as fh:
            fh.write(stext)
    winst = sweep_instantiations(kind)
    winc = os.path.join(CSRC, "sbf_sweep_list.inc")
    wtext = "".join(f"SBF_Z({r}, {p})\n" for r, p in winst)
    if not os.path.exists(winc) or open(winc).read() != wtext:
        with open(winc, "w") as fh:
            fh.write(wtext)
    jobs_list = [(os.path.join(CSRC, s), os.path.join(obj_dir, s.replace(".cu", ".o")), defs)
                 for s in SOURCES]
    for r, p in winst:
        jobs_list.append((os.path.join(CSRC, "sbf_sweep_inst.cu"),
                          os.path.join(obj_dir, f"sweep_r{r}_p{p}.o"),
                          defs + [f"-DSBF_R={r}", f"-DSBF_P={p}"]))
    for r, p in sinst:
        jobs_list.append((os.path.join(CSRC, "sbf_split_inst.cu"),
                          os.path.join(obj_dir, f"split_r{r}_p{p}.o"),
                          defs + [f"-DSBF_R={r}", f"-DSBF_P={p}"]))
    for r, p, m in inst:
        jobs_list.append((os.path.join(CSRC, "sbf_terms_inst.cu"),
                          os.path.join(obj_dir, f"terms_r{r}_p{p}_m{m}.o"),
                          defs + [f"-DSBF_R={r}", f"-DSBF_P={p}", f"-DSBF_M={m}"]))
    jobs = jobs or max(1, os.cpu_count() or 1)
    failed = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        for obj, rc, out in ex.map(_compile, jobs_list):
            if rc != 0:
                failed.append((obj, out))
            elif verbose and out.strip():
                print(out)
    if failed:
        for obj, out in failed:
            sys.stderr.write(f"--- {obj}\n{out}\n")
        raise RuntimeError(f"nvcc failed for {len(failed)} object(s)")
    objs = [j[1] for j in jobs_list]
    if not _newer(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError("link failed:\n" + p.stdout + p.stderr)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    g = ap.add_mutually_exclusive_group()
    g.add_argument("--full", action="store_true")
    g.add_argument("--min", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--variant", default=None, help="experimental build tag")
    ap.add_argument("-D", dest="defs", action="append", default=[], help="extra macro (NAME=VALUE)")
    a = ap.parse_args()
    print(build("min" if a.min else "full", a.j, a.v, a.variant, ["-D" + d for d in a.defs]))
