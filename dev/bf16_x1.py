import sys, math, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import golden_forward
from oracle import flame_oracle as orc
def bf(x): return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).to(torch.float64).numpy()
def fwd(hist, cand, params, cfg, R):
    nh = cfg.hidden_dim // cfg.head_dim
    subs = orc.split_sequence(hist, cfg.num_blocks)
    outs = []
    for sub, blk in zip(subs, params.blocks):
        lay = blk.layers[0]; h = sub.shape[0]
        x = np.concatenate([sub, cand])
        y = R("y", orc.layer_norm(x, lay.ln1_scale, lay.ln1_shift))
        W = lambda w: R("w", w)
        q = R("qkv", y[h:] @ W(lay.w_q)); k = R("qkv", y @ W(lay.w_k)); v = R("qkv", y @ W(lay.w_v))
        H_ = lambda t: t.reshape(t.shape[0], nh, -1).transpose(1, 0, 2)
        qh, kh, vh = H_(q), H_(k), H_(v)
        # attention with P rounded
        scale = 1/(blk.temperature*math.sqrt(cfg.head_dim))
        s_self = np.einsum("hcd,hcd->hc", qh, kh[:, h:]) * scale
        s = (qh @ kh[:, :h].transpose(0, 2, 1)) * scale
        m = np.maximum(s.max(axis=2), s_self)
        w = np.exp(s - m[..., None]); ws = np.exp(s_self - m)
        z = w.sum(axis=2) + ws
        o = R("p", w) @ vh[:, :h] + ws[..., None] * vh[:, h:]
        o = o / z[..., None]
        oc = R("ao", o.transpose(1, 0, 2).reshape(len(cand), -1))
        xc = R("x1", x[h:] + oc @ W(lay.w_o))
        y2 = R("y2", orc.layer_norm(xc, lay.ln2_scale, lay.ln2_shift))
        hf = R("hf", orc.gelu(y2 @ W(lay.w1) + lay.b1))
        outs.append(xc + hf @ W(lay.w2) + lay.b2)
    fz = R("fz", orc.gated_fusion(outs, params))
    he = R("he", orc.gelu(fz @ R("w", params.expert_w1) + params.expert_b1))
    return orc.sigmoid(he @ params.expert_w2 + params.expert_b2)
name = sys.argv[1]
cfg, params, hist, cand, blob = golden_forward(name)
ref = blob["scores"]
hist_b, cand_b = bf(hist), bf(cand)
points = ["w", "y", "qkv", "p", "ao", "y2", "hf", "fz", "he", "x1"]
def run(active, inputs_bf=True):
    R = lambda tag, x: bf(x) if tag in active else x
    return np.abs(fwd(hist_b if inputs_bf else hist, cand_b if inputs_bf else cand, params, cfg, R) - ref).max()
print(name, "inputs only", run(set()))
print(name, "inputs+w", run({"w"}))
for p in points[1:]:
    print(name, f"inputs+w+{p}", run({"w", p}))
print(name, "all", run(set(points)))
print(name, "all but fz,he", run(set(points) - {"fz", "he"}))

dev_now = {"w", "y", "qkv", "p", "ao", "y2", "hf"}   # device rounding points today (fz/he are split/fp32)
print(name, "device today (inputs fp32)", run(dev_now, inputs_bf=False))
print(name, "device + bf16 X1 residual", run(dev_now | {"x1"}, inputs_bf=False))
