"""Build the in-tree CUDA library ``libnlk_b200.so`` for sm_100a.

Every ``csrc/*.cu`` translation unit is compiled in parallel with nvcc
(``-gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false``) and linked
into one shared library next to this file.  ``-fmad=false`` is load-bearing:
the reference rounds every operation separately (numpy, CPython), so the
kernels only fuse where the reference's BLAS does (explicit ``fma()`` calls).
Objects are rebuilt only when a source or header is newer.

    python -m paper_2403_16341_b200.build [--force] [--verbose]
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libnlk_b200.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-I", CSRC, "-I", INCLUDE,
              "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc():
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build")
    return path


def _newest_header():
    hs = (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.inc"))
          + glob.glob(os.path.join(INCLUDE, "*.h")))
    return max(os.path.getmtime(h) for h in hs) if hs else 0.0


def _compile(src, force, verbose, obj_dir=OBJ, defines=(), xptxas=()):
    obj = os.path.join(obj_dir, os.path.basename(src).replace(".cu", ".o"))
    log = obj.replace(".o", ".ptxas.log")
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(src), _newest_header())):
        return obj, None
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *source_flags(src), *[f"-D{d}" for d in defines],
           *[a for x in xptxas for a in ("-Xptxas", x)], "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-4000:]}")
    return obj, log


def source_flags(src):
    """Per-file nvcc flags from `// nlk-build: <flags>` lines in the source
    (e.g. a ptxas option measured better for the one kernel in that file)."""
    flags = []
    with open(src) as fh:
        for line in fh:
            if line.startswith("// nlk-build:"):
                flags += line.split(":", 1)[1].split()
    return flags


def source_files():
    """The files the library is built from (build-id inputs)."""
    fs = []
    for pat in ("*.cu", "*.cuh", "*.inc", "*.h"):
        fs += glob.glob(os.path.join(CSRC, pat))
    fs += glob.glob(os.path.join(INCLUDE, "*.h"))
    return sorted(fs)


def source_build_id():
    """First 16 hex digits of SHA-256 over (relative name, contents) of every
    source file, sorted by name (nlk_build_id() of a library built from them)."""
    import hashlib
    h = hashlib.sha256()
    for f in source_files():
        h.update(os.path.relpath(f, ROOT).encode() + b"\0")
        with open(f, "rb") as fh:
            h.update(fh.read())
        h.update(b"\0")
    return h.hexdigest()[:16]


def _build_id_object(obj_dir, defines):
    """Compile the one-function TU that carries the build id (+ variant
    defines, so a variant library reports what it was built with)."""
    bid = source_build_id() + ("+" + ",".join(defines) if defines else "")
    src = os.path.join(obj_dir, "nlk_build_id.cu")
    obj = os.path.join(obj_dir, "nlk_build_id.o")
    text = ('#include "nlk_b200.h"\n'
            f'extern "C" NLK_API const char* nlk_build_id(void) {{ return "{bid}"; }}\n')
    if not (os.path.exists(src) and open(src).read() == text and os.path.exists(obj)):
        with open(src, "w") as fh:
            fh.write(text)
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-4000:]}")
    return obj


def build(force=False, verbose=False, jobs=None, tag=None, defines=(), only=None, xptxas=()):
    """Compile and link; ``tag``/``defines`` make a variant library
    ``libnlk_b200_<tag>.so`` (objects in ``_obj_<tag>``) for A/B timing.
    ``only`` (variants): recompile just the sources whose name contains one
    of these substrings and link the default build's objects for the rest."""
    obj_dir, lib = (OBJ, LIB) if not tag else (OBJ + "_" + tag, LIB.replace(".so", f"_{tag}.so"))
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or os.cpu_count() or 4
    mine = [s for s in srcs if not only or any(k in os.path.basename(s) for k in only)]
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose, obj_dir, defines, xptxas), mine))
    objs = [o for o, _ in results]
    if only:  # the rest from the default build (must be current)
        objs += [os.path.join(OBJ, os.path.basename(s).replace(".cu", ".o")) for s in srcs
                 if s not in mine]
    objs += [_build_id_object(obj_dir, list(defines) + [f"ptxas:{x}" for x in xptxas])]
    if (force or not os.path.exists(lib)
            or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs)):
        cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("-j", "--jobs", type=int, default=None)
    ap.add_argument("--tag", default=None, help="variant name (separate objects and .so)")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra -D for nvcc")
    ap.add_argument("--only", action="append", default=None,
                    help="variant: recompile only sources containing this substring")
    ap.add_argument("--xptxas", action="append", default=[],
                    help="variant: extra ptxas option (e.g. --register-usage-level=8)")
    a = ap.parse_args(argv)
    if (a.defines or a.xptxas) and not a.tag:
        ap.error("-D / --xptxas build variants and need --tag")
    print(build(a.force, a.verbose, a.jobs, a.tag, a.defines, a.only, a.xptxas))


if __name__ == "__main__":
    sys.exit(main())
