mkdir -p gpurun_out
timeout 900 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
cat gpurun_out/sweep.jsonl; tail -3 gpurun_out/sweep.err
cat > /tmp/san.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2406_16747_b200 import ops
dev = torch.device("cuda", 0)
for D in (64, 128):
    L, H = 600, 2
    g = torch.Generator(device=dev); g.manual_seed(1)
    q, k, v, do = (torch.randn((1, L, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    u = torch.randn((1, L), generator=g, device=dev, dtype=torch.float64) + 0.01 * torch.arange(L, device=dev)
    cfg = ops.AttnConfig(k=100.5, window=40)
    o, lse, sel = ops.attn_fwd(q, k, v, u, cfg)
    ops.attn_bwd(q, k, v, o, do, lse, u, sel, cfg)
    c = ops.DecodeCache(1, H, D, cfg, max_len=L)
    c.prefill(k[:, :500].contiguous(), v[:, :500].contiguous(), u[:, :500].contiguous())
    for i in range(500, 510):
        c.step(q[:, i].contiguous(), k[:, i].contiguous(), v[:, i].contiguous(), u[:, i].contiguous())
torch.cuda.synchronize()
print("sanitized run ok")
PY
for tool in memcheck synccheck racecheck; do timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.log; done
