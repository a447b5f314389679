"""Build libwavestep.so in-tree for sm_100a (``python -m paper_1308_1464_b200.build``).

Flags that matter for parity: ``--fmad=false`` (no contraction of a*b+c into
an FMA, so every product and sum rounds like numpy), ``-prec-div=true
-prec-sqrt=true -ftz=false`` (IEEE division / square root, denormals kept).
The fp32 throughput mode's units (``ws_inst_fast_*.cu``) use FAST_FLAGS.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
SOURCES = [CSRC / "wavestep.cu"] + sorted(CSRC.glob("ws_inst_*.cu"))
OUT = HERE / "_lib" / "libwavestep.so"
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [HERE.parent / "include" / "wavestep.h", Path(__file__).resolve()]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC",
]

# the fp32 throughput mode's units (ws_inst_fast_*.cu, WS_FP32_FAST): FMA
# contraction, the approximate division / square root and denormals flushed
# to zero (division = MUFU.RCP + FMUL with one range fix-up, square root and
# reciprocal = one MUFU); their parity is a stated bound against fp64, not
# bits
FAST_FLAGS = [{"--fmad=false": "--fmad=true", "-prec-div=true": "-prec-div=false",
               "-prec-sqrt=true": "-prec-sqrt=false", "-ftz=false": "-ftz=true"}.get(f, f)
              for f in NVCC_FLAGS]


# per-unit additions (measured per kernel, profiles/r2_s6_ab.md): ptxas'
# register-usage level 2 (default 5) for the three-wave fp64 shallow-water
# kernels only
UNIT_FLAGS = {"ws_inst_shallow_roe.cu": ["-Xptxas", "--register-usage-level=2"]}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


# the checked variant (-DWS_CHECKED=1): device index checks, per-cell write
# counts and NaN canaries; the GPU tests load it with WAVESTEP_LIB
CHECKED_OUT = HERE / "_lib" / "checked" / "libwavestep.so"


def up_to_date(out: Path | None = None) -> bool:
    out = OUT if out is None else out
    if not out.exists():
        return False
    t = out.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS)


def build_all(force: bool = False, verbose: bool = False) -> Path:
    """The product library and its checked variant (both in-tree, sm_100a)."""
    from concurrent.futures import ThreadPoolExecutor
    jobs = [lambda: build(force, verbose)]
    if force or not up_to_date(CHECKED_OUT):
        jobs.append(lambda: build(True, verbose, ("WS_CHECKED=1",), CHECKED_OUT))
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        outs = [f.result() for f in [ex.submit(j) for j in jobs]]
    return outs[0]


def build(force: bool = False, verbose: bool = False, defines: tuple = (),
          out: Path | None = None) -> Path:
    """Compile every translation unit (in parallel) and link libwavestep.so.

    ``defines`` / ``out``: an experimental variant (e.g. WS_LB3=0) built into
    its own directory; load it with WAVESTEP_LIB=<out>."""
    if out is not None:
        return _build(Path(out), verbose, defines)
    if not force and not defines and up_to_date():
        return OUT
    return _build(OUT, verbose, defines)


def _build(OUT: Path, verbose: bool, defines: tuple) -> Path:
    from concurrent.futures import ThreadPoolExecutor
    OUT.parent.mkdir(parents=True, exist_ok=True)
    objdir = OUT.parent / "obj"
    objdir.mkdir(exist_ok=True)
    log = OUT.parent / "build.log"

    def compile_one(src: Path):
        obj = objdir / (src.stem + ".o")
        flags = FAST_FLAGS if src.name.startswith("ws_inst_fast_") else NVCC_FLAGS
        extra = os.environ.get("WS_NVCC_EXTRA", "").split()   # experiments only
        cmd = [nvcc(), *flags, *UNIT_FLAGS.get(src.name, []), *extra, *(f"-D{d}" for d in defines),
               "-Xptxas", "-v", "-c",
               "-o", str(obj), str(src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, res

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    text = []
    for src, obj, cmd, res in results:
        text.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            log.write_text("\n".join(text))
            sys.stderr.write(res.stderr[-4000:])
            raise RuntimeError(f"nvcc failed on {src.name} ({res.returncode}); see {log}")
    tmp = OUT.with_suffix(".so.tmp")
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
            "-Xcompiler", "-fPIC", "-o", str(tmp)] + [str(r[1]) for r in results]
    res = subprocess.run(link, capture_output=True, text=True)
    text.append(" ".join(link) + "\n" + res.stdout + res.stderr)
    log.write_text("\n".join(text))
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError(f"link failed ({res.returncode}); see {log}")
    os.replace(tmp, OUT)
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    # python -m paper_1308_1464_b200.build [--force] [--define X=1 ...] [--out path.so]
    a = sys.argv[1:]
    defs = tuple(a[i + 1] for i, x in enumerate(a) if x == "--define")
    out = a[a.index("--out") + 1] if "--out" in a else None
    if defs or out:
        build(force="--force" in a, verbose=True, defines=defs, out=out)
    else:
        build_all(force="--force" in a, verbose=True)
