import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
g = torch.Generator(device="cuda").manual_seed(3)
for rows, vocab, d in [(339, 1000, 64), (300, 1000, 64), (4096, 32000, 512)]:
    h = torch.randn(rows, d, device=dev, generator=g).bfloat16()
    W = (torch.randn(vocab, d, device=dev, generator=g) / 8).bfloat16()
    bias = torch.zeros(vocab, device=dev)
    logits = torch.empty(rows, vocab, device=dev, dtype=torch.bfloat16)
    labels = torch.randint(0, vocab, (rows,), device=dev, generator=g, dtype=torch.int32)
    loss = torch.empty(rows, device=dev)
    lsum = torch.zeros(1, device=dev)
    ops.gemm(h, W, logits, epilogue=ops.EPI_BF16, bias=bias)
    ref_logits = logits.clone()
    ops.xent(logits, labels, logits, loss, 1.0 / rows, loss_sum=lsum)
    torch.cuda.synchronize()
    lf = ref_logits.float().requires_grad_(True)
    ce = torch.nn.functional.cross_entropy(lf, labels.long(), reduction="sum") / rows
    ce.backward()
    err = (logits.float() - lf.grad).abs().max().item()
    print(rows, vocab, "nan", torch.isnan(logits).sum().item(), "maxerr", err, "loss", lsum.item(), ce.item())
