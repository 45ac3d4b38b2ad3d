"""BASELINE.json configs[4]: sweep k x L at d=128, w=512 (bf16 fwd+bwd, tensor-core path,
recency scores) and report time, tokens/s and the fraction of the sustained bf16 peak on the
algorithmic FLOPs (4+8)*d*N_att. H=8, B=1 per point (units are independent (b, h) pairs, so
throughput per unit is what the sweep maps). Writes one line per point (JSON) to stdout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2406_16747_b200 import ops  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    _, _, tf_sus, _ = bench.peaks()
    H, d, w = 8, 128, 512
    gather = "--gather" in sys.argv  # the CUDA-core gather path (force_gather) for the regime map
    Ls = (4096, 16384) if gather else (4096, 16384, 65536)
    for L in Ls:
        for k in (64.0, 256.0, 1024.0, 4096.0):
            if k + w >= L:
                continue
            g = torch.Generator(device=dev)
            g.manual_seed(L + int(k))
            q, kk, v, do = (torch.randn((1, L, H, d), generator=g, device=dev).to(torch.bfloat16)
                            for _ in range(4))
            u = (torch.randn((1, L), generator=g, device=dev, dtype=torch.float64)
                 + 0.01 * torch.arange(1, L + 1, device=dev, dtype=torch.float64))
            cfg = ops.AttnConfig(k=k, window=w, force_gather=gather)
            ws = ops.bwd_workspace(q, cfg)

            def step():
                sel = ops.select(u, cfg, heads=H, head_dim=d, dtype=torch.bfloat16)
                o, lse, _ = ops.attn_fwd(q, kk, v, u, cfg, sel=sel)
                ops.attn_bwd(q, kk, v, o, do, lse, u, sel, cfg, ws=ws)

            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 5
            e0.record()
            for _ in range(n):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            natt = bench.n_att(L, k, w)
            fl = 12.0 * d * natt * H
            print(json.dumps({"path": "gather" if gather else "tcgen05", "L": L, "k": k, "w": w, "H": H,
                              "d": d, "ms": round(ms, 3),
                              "tokens_per_s": round(L / (ms / 1e3)), "tflops": round(fl / ms / 1e9, 1),
                              "frac_of_sustained": round(fl / ms / 1e9 / tf_sus, 3),
                              "keys_per_query": round(natt / L, 1)}), flush=True)
            del q, kk, v, do, u, ws
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
