import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2509_22681_b200 as fb
from oracle import flame_oracle as orc
def run(cfg, H, C, seed=0, prec="bf16"):
    params = fb.init_params(cfg)
    rng = np.random.default_rng(seed)
    hist = rng.uniform(-1, 1, (H, cfg.hidden_dim)); cand = rng.uniform(-1, 1, (C, cfg.hidden_dim))
    t0 = time.time()
    got = fb.model_forward(hist, cand, params, cfg, precision=prec)
    t1 = time.time()
    ref = orc.model_forward(hist, cand, params, cfg)
    err = np.abs(got - ref).max()
    print(f"{prec} d={cfg.hidden_dim} dh={cfg.head_dim} Nb={cfg.num_blocks} L={cfg.layers_per_block} H={H} C={C}: maxabs={err:.3e} ({t1-t0:.2f}s)", flush=True)
    return err
cfg1 = fb.ModelConfig(64, 16, 2, 1, 256, 2, 256, 64, seed=0)
for prec in ("fp32", "bf16"):
    run(cfg1, 256, 64, prec=prec)
    run(fb.ModelConfig(16, 4, 2, 2, 24, 3, 64, 32, seed=11), 16, 5, prec=prec)
    run(fb.ModelConfig(256, 64, 4, 1, 1024, 2, 1024, 256, seed=0), 1024, 256, prec=prec)
    run(fb.ModelConfig(64, 16, 2, 2, 128, 2, 512, 300, seed=3), 512, 300, prec=prec)
    run(fb.ModelConfig(64, 16, 2, 1, 256, 2, 256, 64, seed=0), 0, 7, prec=prec)
