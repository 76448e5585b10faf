"""How many (candidate, step, GPU) gathers the K5 step floors skip on a bench
trace: per lane and per warp of 32 steps (the kernel's warp-uniform branch),
with the per-step level min_g s_g(h) the kernel uses and with per-GPU levels.

    python tools/floor_stats.py [--config deepseek-v3] [--cands 256] [--layers 2]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19945_b200 as gem  # noqa: E402
from paper_2605_19945_b200 import _device, ingest  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="deepseek-v3")
    ap.add_argument("--cands", type=int, default=256)
    ap.add_argument("--layers", type=int, default=2)
    a = ap.parse_args()
    L, N, k, E, B, G, _ = bench.CONFIGS[a.config]
    planted = {} if E >= 16 else {"consistent": 2, "num_groups": 1}
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0,
                                **planted)
    ids = ingest.generate_topk_ids(spec, dtype=torch.int16)
    hist = ingest.ids_to_histograms(ids, B, E).hist[: a.layers]  # [l, T, E] int32
    del ids
    prof = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64,
                                                         max_tokens=B * k, rng_seed=0))
    dc = _device.DeviceCurves.from_profile(prof)
    lut = dc.lut(B * k)  # [G, nmax+1] fp64
    rng = np.random.default_rng(0)
    base = np.repeat(np.arange(G, dtype=np.int64), E // G)
    res = {}
    for l in range(a.layers):
        h = hist[l].double()  # [T, E]
        T = h.shape[0]
        hm = hist[l].max(dim=1).values.long()  # [T]
        v = lut[:, hm].min(dim=0).values  # [T]
        sg = torch.stack([torch.searchsorted(lut[g].contiguous(), v, right=True) - 1 for g in range(G)])  # [G, T]
        smin = sg.min(dim=0).values
        lane_k = lane_g = warp_k = warp_g = 0
        for c in range(a.cands):
            oh = torch.zeros((E, G), dtype=torch.float64, device="cuda")
            oh[torch.arange(E), torch.from_numpy(rng.permutation(base)).cuda()] = 1
            loads = (h @ oh).long()  # [T, G]
            above_k = loads > smin[:, None]
            above_g = loads > sg.T
            lane_k += above_k.sum().item()
            lane_g += above_g.sum().item()
            Tw = T // 32 * 32
            warp_k += above_k[:Tw].view(-1, 32, G).any(dim=1).sum().item() * 32
            warp_g += above_g[:Tw].view(-1, 32, G).any(dim=1).sum().item() * 32
        tot = a.cands * T * G
        res[l] = {"gathered_lane_minlevel": lane_k / tot, "gathered_lane_pergpu": lane_g / tot,
                  "gathered_warp_minlevel": warp_k / tot, "gathered_warp_pergpu": warp_g / tot,
                  "hmax_median": hm.median().item(), "smin_median": smin.median().item(),
                  "sg_median_range": [sg.median(dim=1).values.min().item(), sg.median(dim=1).values.max().item()]}
    print(json.dumps({"config": a.config, "G": G, "layers": res}))


if __name__ == "__main__":
    main()
