"""Per-k-block pipeline timeline of CTA 0 for one GEMM launch (clock64):
when the producer refills each stage and when the MMA warp gets each stage."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import _native, ops
dev = torch.device("cuda:0")
L = _native.lib()
m, n, k = (int(x) for x in sys.argv[1:4])
A = torch.randn(m, k, device=dev).bfloat16()
B = torch.randn(n, k, device=dev).bfloat16()
D = torch.zeros(m, n, device=dev, dtype=torch.bfloat16)
buf = torch.zeros(8 * 148 + 1024, dtype=torch.int64, device=dev)
for _ in range(5):
    ops.gemm(A, B, D, epilogue=ops.EPI_BF16)
torch.cuda.synchronize()
L.mm_gemm_trace(buf.data_ptr())
ops.gemm(A, B, D, epilogue=ops.EPI_BF16)
torch.cuda.synchronize()
L.mm_gemm_trace(None)
t = buf[8 * 148:8 * 148 + 256].cpu().numpy()
prod, mma = t[:128], t[128:]
base = min(x for x in np.concatenate([prod, mma]) if x > 0)
p = [(x - base) for x in prod if x > 0]
q = [(x - base) for x in mma if x > 0]
print("producer refill (cycles):", p[:40])
print("mma gets stage (cycles): ", q[:40])
print("mma deltas:", np.diff(q)[:40].tolist())
t2 = buf[8 * 148 + 512:8 * 148 + 768].cpu().numpy()
iss, com = t2[:128], t2[128:]
q = np.array([x for x in mma if x > 0])
iss = np.array([x for x in iss if x > 0]); com = np.array([x for x in com if x > 0])
print("issue MMAs (cycles after full wait):", (iss - q[:len(iss)])[:20].tolist())
print("commit   (cycles after MMAs issued):", (com - iss[:len(com)])[:20].tolist())
