"""Build a tuning variant of libmmb200.so with extra -D flags for gemm.cu:
    python tools/build_variant.py NAME -DMM_GEMM_EPI_WARPS=4 ...
-> build/variants/NAME/libmmb200.so (load with MM_LIB_VARIANT=NAME)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import build_native as B
name, flags = sys.argv[1], sys.argv[2:]  # e.g. -DMM_GEMM_KB_TRACE for tools/gemm_kbtrace.py
out = os.path.join(B.ROOT, "build", "variants", name)
os.makedirs(out, exist_ok=True)
B.build()
nccl_inc, nccl_lib = B.nccl_dirs()
obj = os.path.join(out, "gemm.cu.o")
cmd = [B._nvcc(), "-c", os.path.join(B.CSRC, "gemm.cu"), "-o", obj, "-O3", "-std=c++17", *B.ARCH,
       "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", B.INCLUDE, "-I", B.CSRC,
       "-I", nccl_inc, "--expt-relaxed-constexpr", *flags]
subprocess.run(cmd, check=True)
objs = [obj] + [os.path.join(B.OBJDIR, f) for f in os.listdir(B.OBJDIR) if f != "gemm.cu.o"]
subprocess.run([B._nvcc(), "-shared", "-o", os.path.join(out, "libmmb200.so"), *objs, *B.ARCH,
                "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl_lib}"], check=True)
print(out)
