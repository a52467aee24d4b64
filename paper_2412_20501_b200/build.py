"""Build libtokenring.so in-tree with nvcc for sm_100a (no JIT cache, so the
built library travels to the GPU box with the repository snapshot).

    python -m paper_2412_20501_b200.build          # incremental
    python -m paper_2412_20501_b200.build --force
    python -m paper_2412_20501_b200.build --experiments
        # A/B build (not the product): + the measured-and-rejected kernel
        # variants of attn_fwd_variants.cu and their TR_ATTN_* run-time
        # switches, -> _variants/libtokenring_exp.so
"""

import argparse
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtokenring.so")
ROOT = os.path.dirname(HERE)

SOURCES = ["capi.cu", "attn_fwd_sm100.cu", "attn_fwd_pair2.cu", "attn_simt.cu",
           "lse_merge.cu", "splitmix.cu", "p2p_flags.cu"]
EXPERIMENT_SOURCES = ["attn_fwd_variants.cu"]
EXP_LIB = os.path.join(HERE, "_variants", "libtokenring_exp.so")
HEADERS = ["tr_ptx.cuh", "tr_internal.h", "attn_common.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.abspath(__file__))
    deps.append(os.path.join(ROOT, "include", "tokenring.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, defines=(), out=None, experiments=False):
    """Compile every .cu and link libtokenring.so (or ``out`` -- tuning
    variants built with extra -D ``defines``).  ``experiments`` adds the
    rejected kernel variants and their run-time switches (never the product)."""
    if experiments:
        defines = tuple(defines) + ("TR_EXPERIMENTS",)
        out = out or EXP_LIB
        os.makedirs(os.path.dirname(out), exist_ok=True)
    lib = out or LIB
    if not force and not defines and not _stale():
        return LIB
    objs = []
    tmp = os.path.join(HERE, "_build", "_".join(d.replace("=", "") for d in defines) or "main")
    os.makedirs(tmp, exist_ok=True)
    nvcc = nvcc_path()
    common = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr",
              *[f"-D{d}" for d in defines]]
    if verbose:
        common += ["-Xptxas", "-v"]
    procs = []
    for src in SOURCES + (EXPERIMENT_SOURCES if experiments else []):
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        objs.append(obj)
        procs.append((src, subprocess.Popen(common + ["-c", os.path.join(CSRC, src), "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode()}")
        if verbose:
            print(out.decode())
    link = [nvcc, *ARCH, "-shared", "-o", lib + ".tmp", *objs]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--out", default=None)
    ap.add_argument("--experiments", action="store_true")
    a = ap.parse_args(argv)
    print(build(force=a.force, verbose=a.verbose, defines=tuple(a.defines), out=a.out,
                experiments=a.experiments))


if __name__ == "__main__":
    sys.exit(main())
