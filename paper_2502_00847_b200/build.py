"""Build libsecpe.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_2502_00847_b200.build          # incremental
    python -m paper_2502_00847_b200.build --clean
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libsecpe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-Xptxas", "-warn-spills"]
SOURCES = ["ntt.cu", "ntt_fused.cu", "ops.cu", "ks.cu", "bconv_tc.cu", "sample.cu", "context.cu", "eval.cu", "plan.cu", "client.cu",
           "encode.cpp", "boot.cpp", "abi.cpp"]


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(HERE, "..", "include", "secpe.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src, hm, obj=OBJ, defines=()):
    s = os.path.join(CSRC, src)
    o = os.path.join(obj, src + ".o")
    if os.path.exists(o) and os.path.getmtime(o) >= max(os.path.getmtime(s), hm):
        return o, None
    cmd = [NVCC] + ARCH + FLAGS + ["-D" + d for d in defines] + ["-x", "cu", "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return o, "%s\n%s\n%s" % (" ".join(cmd), r.stdout, r.stderr)
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return o, None


def build(clean=False, verbose=False, variant=None, defines=()):
    """Build libsecpe.so; `variant` (development experiments) builds libsecpe_<variant>.so with extra
    -D defines in its own object directory."""
    obj = OBJ if variant is None else os.path.join(OBJ, "v_" + variant)
    lib = LIB if variant is None else os.path.join(HERE, "libsecpe_%s.so" % variant)
    if clean and os.path.isdir(obj):
        shutil.rmtree(obj)
    os.makedirs(obj, exist_ok=True)
    hm = _headers_mtime()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        res = list(ex.map(lambda s: _compile(s, hm, obj, defines), SOURCES))
    errs = [e for _, e in res if e]
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    objs = [o for o, _ in res]
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lquadmath", "-lcudart"]
        subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    # python -m paper_2502_00847_b200.build [--clean] [--variant NAME DEF=V ...]
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        print(build(clean="--clean" in args, variant=args[i + 1], defines=args[i + 2:]))
    else:
        print(build(clean="--clean" in args))
