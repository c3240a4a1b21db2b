"""Build a tuning variant of libmmb200.so:
    python tools/build_variant.py NAME [--all] [-DFLAG ...] [file.cu=/path/to/alt.cu ...]
-D flags apply to gemm.cu and every substituted source (e.g. -DMM_GEMM_KB_TRACE),
or with --all to every CUDA source (e.g. the bounds-checked debug build:
`dbg --all -DMM_DEBUG_BOUNDS`);
file.cu=path substitutes a source (e.g. an older kernel from `git show`).
-> build/variants/NAME/libmmb200.so (load with MM_LIB_VARIANT=NAME)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import build_native as B
name = sys.argv[1]
all_src = "--all" in sys.argv[2:]
flags = [a for a in sys.argv[2:] if a.startswith("-") and a != "--all"]
subs = dict(a.split("=", 1) for a in sys.argv[2:] if "=" in a and not a.startswith("-"))
out = os.path.join(B.ROOT, "build", "variants", name)
os.makedirs(out, exist_ok=True)
B.build()
nccl_inc, nccl_lib = B.nccl_dirs()
objs = []
for f in sorted(os.listdir(B.OBJDIR)):
    src = f[:-2]  # strip .o
    if (src == "gemm.cu" or (all_src and src.endswith(".cu"))) and flags or src in subs:
        obj = os.path.join(out, f)
        path = subs.get(src, os.path.join(B.CSRC, src))
        cmd = [B._nvcc(), "-c", path, "-o", obj, "-O3", "-std=c++17", *B.ARCH, "-lineinfo",
               "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", B.INCLUDE, "-I", B.CSRC,
               "-I", nccl_inc, "--expt-relaxed-constexpr", *flags]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    else:
        objs.append(os.path.join(B.OBJDIR, f))
subprocess.run([B._nvcc(), "-shared", "-o", os.path.join(out, "libmmb200.so"), *objs, *B.ARCH,
                "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl_lib}"], check=True)
print(out)
