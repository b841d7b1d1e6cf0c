"""Scores of a few shapes with the current FLAME_FUSED_ATTN setting, saved for an
A/B against the unfused path: python dev/fused_ab.py OUT.npz"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2509_22681_b200 as fb

CASES = {"d768_hb256": (768, 64, 2, 1, 1536, 2, 512, 256), "d512_hb682": (512, 64, 2, 1, 1024, 2, 1364, 256),
         "d128_hb300": (128, 64, 1, 1, 256, 2, 300, 100), "d256_hb130": (256, 64, 2, 1, 512, 2, 260, 300)}
out = {}
for name, (d, dh, nb, L, f, t, H, C) in CASES.items():
    cfg = fb.ModelConfig(d, dh, nb, L, f, t, H, C, seed=3)
    p = fb.init_params(cfg)
    rng = np.random.default_rng(1)
    s = fb.model_forward(rng.uniform(-1, 1, (H, d)), rng.uniform(-1, 1, (C, d)), p, cfg)
    out[name] = s
    print(name, "nan" if np.isnan(s).any() else "ok", float(np.nanmax(s)))
np.savez(sys.argv[1], **out)
