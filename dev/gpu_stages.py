import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2509_22681_b200 as fb
from oracle import flame_oracle as orc
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
cfg = fb.ModelConfig(64, 16, 2, 1, 256, 2, 256, 64, seed=0)
params = fb.init_params(cfg)
rng = np.random.default_rng(0)
H, C = 256, 64
hist = rng.uniform(-1, 1, (H, 64)); cand = rng.uniform(-1, 1, (C, 64))
eng = fb.get_engine(params, cfg, prec)
hb_bkt, c_bkt = eng.bucket(H, C)
ex = eng.executor(1, hb_bkt, c_bkt)
got = ex.score([(hist, cand)], graph=False)[0]
ref = orc.model_forward(hist, cand, params, cfg)
print("final maxabs", np.abs(got - ref).max())
G, D, DA, F = 2, 64, 4 * 64, 256
hb = H // G
rows = hb_bkt + c_bkt
dt = np.float32
Eh = ex.read_workspace("Eh", (G, hb_bkt, D))
Ec = ex.read_workspace("Ec", (c_bkt, D))
print("Eh err", np.abs(Eh[:, :hb] - hist.reshape(G, hb, 64)).max(), "Ec err", np.abs(Ec[:C] - cand).max())
if prec == "fp32":
    qkv = ex.read_workspace("qkv", (G, rows, 3 * DA))
    attn = ex.read_workspace("attn", (G, rows, DA))
    x1 = ex.read_workspace("x1", (G, rows, D))
    xo = ex.read_workspace("xout", (G, rows, D))
    fz = ex.read_workspace("fused", (c_bkt, D))
    nh = 4
    def padheads(x):  # (T, 64) -> (T, 256) head h at h*64
        out = np.zeros((x.shape[0], DA))
        for h in range(nh): out[:, h*64:h*64+16] = x[:, h*16:(h+1)*16]
        return out
    outs = []
    for g in range(G):
        blk = params.blocks[g]; lay = blk.layers[0]
        sub = hist[g*hb:(g+1)*hb]
        x = np.concatenate([sub, cand])
        y = orc.layer_norm(x, lay.ln1_scale, lay.ln1_shift)
        k = y @ lay.w_k; v = y @ lay.w_v; q = y[hb:] @ lay.w_q
        print(f"g{g} K hist err", np.abs(qkv[g, :hb, DA:2*DA] - padheads(k[:hb])).max(),
              "V hist err", np.abs(qkv[g, :hb, 2*DA:] - padheads(v[:hb])).max())
        print(f"g{g} Q cand err", np.abs(qkv[g, hb_bkt:hb_bkt+C, :DA] - padheads(q)).max(),
              "K cand err", np.abs(qkv[g, hb_bkt:hb_bkt+C, DA:2*DA] - padheads(k[hb:])).max())
        qh = q.reshape(C, nh, 16).transpose(1, 0, 2); kh = k.reshape(-1, nh, 16).transpose(1, 0, 2); vh = v.reshape(-1, nh, 16).transpose(1, 0, 2)
        oc = orc.sumi_candidates(qh, kh, vh, hb, 1.0)
        ocm = oc.transpose(1, 0, 2).reshape(C, 64)
        print(f"g{g} attn err", np.abs(attn[g, hb_bkt:hb_bkt+C] - padheads(ocm)).max())
        xc = cand + ocm @ lay.w_o
        print(f"g{g} x1 err", np.abs(x1[g, hb_bkt:hb_bkt+C] - xc).max())
        o = orc.block_forward(sub, cand, blk, nh)
        outs.append(o)
        print(f"g{g} xout err", np.abs(xo[g, hb_bkt:hb_bkt+C] - o).max())
    print("fused err", np.abs(fz[:C] - orc.gated_fusion(outs, params)).max())
