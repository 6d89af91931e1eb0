"""Build liboccx.so for sm_100a, in-tree (python -m paper_1701_08547_b200.build).

nvcc cross-compiles without a GPU.  Flags: -gencode arch=compute_100a,
code=sm_100a -lineinfo -O3; the feature kernel is compiled with
-fmad=false so no multiply-add contraction changes a rounding step
(DESIGN.md §5).  Object files are cached by source mtime.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liboccx.so")
BUILD = os.path.join(HERE, "_objs")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "-cudart", "shared"]
CXX = os.environ.get("CXX", "g++")
CXX_SOURCES = {"occx_sass.cpp": []}     # host-only C++ (tokenizer)
# + csrc/occx_host.cpp: CPython extension _occx_host (plan packing, decoding)
SOURCES = {
    "occx_capi.cu": [],
    "occx_score.cu": [],
    "occx_mix.cu": [],
    "occx_feat.cu": ["-fmad=false"],
}


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, timing: bool = False, variant: str = "",
          defs: tuple = ()) -> str:
    """Compile the stale sources (in parallel) and link liboccx.so.
    ``timing``: the instrumented K2 build (-DOCCX_K2_TIMING: per-CTA
    globaltimer spans and slow-path counters, scripts/k2_profile.py) into
    _objs_timing/liboccx_timing.so -- experiments only, never loaded by
    the package unless OCCX_LIB names it."""
    # experiment builds (never loaded unless OCCX_LIB names them): the
    # instrumented K2 (timing) or a named variant with extra -D flags
    tag = "_timing" if timing else (f"_{variant}" if variant else "")
    build_dir = BUILD + tag
    out = os.path.join(build_dir, f"liboccx{tag}.so") if tag else OUT
    defs = (["-DOCCX_K2_TIMING"] if timing else []) + [f"-D{d}" for d in defs]
    os.makedirs(build_dir, exist_ok=True)
    header_deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
                   if f.endswith((".cuh", ".h"))]
    header_deps += [os.path.join(os.path.dirname(HERE), "include", "occx.h"), __file__]
    objs, jobs = [], []
    for src, extra in SOURCES.items():
        path = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        if _stale(obj, [path] + header_deps):
            jobs.append((src, [NVCC, *ARCH, *COMMON, *defs, *extra, "-c", path, "-o", obj]))
    for src, extra in CXX_SOURCES.items():
        path = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, src.replace(".cpp", ".o"))
        objs.append(obj)
        if _stale(obj, [path] + header_deps):
            jobs.append((src, [CXX, "-O3", "-std=c++17", "-fPIC", "-Wall", "-c", path,
                               "-o", obj, *extra]))
    procs = [(src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                    text=True)) for src, cmd in jobs]
    failed = []
    for src, pr in procs:
        log, _ = pr.communicate()
        if verbose or pr.returncode:
            sys.stderr.write(log)
        if pr.returncode:
            failed.append(src)
    if failed:
        raise RuntimeError(f"compile failed on {', '.join(failed)}")
    if not tag:           # the native host module (CPython extension, csrc/occx_host.cpp)
        import sysconfig
        ext = os.path.join(HERE, "_occx_host" + sysconfig.get_config_var("EXT_SUFFIX"))
        src = os.path.join(CSRC, "occx_host.cpp")
        if _stale(ext, [src, __file__]):
            r = subprocess.run([CXX, "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall",
                                "-I" + sysconfig.get_paths()["include"], src, "-o", ext],
                               capture_output=True, text=True)
            if r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError("compile failed on occx_host.cpp")
    if _stale(out, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", out, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"link of {os.path.basename(out)} failed")
    return out


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    dd = tuple(a.split("=", 1)[1] for a in sys.argv if a.startswith("--define="))
    print(build(verbose="-v" in sys.argv, timing="--timing" in sys.argv, variant=var, defs=dd))
