"""Host API mirror: ModelConfig / init_params / FLMP files are byte-identical
with the reference (golden sha256 + a reference-written FLMP image)."""

import hashlib

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from conftest import FORWARD_CASES, golden_forward, load_golden


@pytest.mark.parametrize("name", FORWARD_CASES)
def test_init_params_bytes_match_reference(name):
    cfg, params, *_ = golden_forward(name)
    g = load_golden("params.npz")
    want = dict(zip(g["sha_names"].tolist(), g["sha_values"].tolist()))[name]
    assert hashlib.sha256(fb.params_to_bytes(params, cfg)).hexdigest() == want


def test_load_reference_flmp_file(tmp_path):
    g = load_golden("params.npz")
    path = tmp_path / "ref.flmp"
    path.write_bytes(g["flmp_tiny"].tobytes())
    cfg, params = fb.load_params(path)
    assert cfg.seed == (1 << 40) + 17 and cfg.layers_per_block == 2
    fresh = fb.init_params(cfg)
    for (na, a), (nb, b) in zip(fb.iter_param_arrays(params), fb.iter_param_arrays(fresh)):
        assert na == nb
        np.testing.assert_array_equal(a, b)
    assert fb.params_to_bytes(params, cfg) == g["flmp_tiny"].tobytes()


def test_flmp_round_trip_and_errors(tmp_path):
    cfg = fb.ModelConfig(16, 4, 2, 1, 24, 3, 64, 32, seed=2**64 - 1)
    p = fb.init_params(cfg)
    path = tmp_path / "x.flmp"
    fb.save_params(p, cfg, path)
    cfg2, p2 = fb.load_params(path)
    assert cfg2 == cfg
    assert fb.params_to_bytes(p2, cfg2) == path.read_bytes()
    raw = path.read_bytes()
    (tmp_path / "bad").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError):
        fb.load_params(tmp_path / "bad")
    (tmp_path / "trail").write_bytes(raw + b"\0" * 8)
    with pytest.raises(ValueError):
        fb.load_params(tmp_path / "trail")


def test_param_stream_order_and_size():
    cfg = fb.ModelConfig(8, 4, 2, 2, 12, 2, 16, 8)
    p = fb.init_params(cfg)
    s = fb.param_stream(p)
    d, f, t = 8, 12, 2
    per_layer = 4 * d * d + 4 * d + d * f + f + f * d + d
    assert s.size == 2 * (2 * per_layer + 1 + 2 * d) + d * f + f + f * t + t
    assert s[0] == p.blocks[0].layers[0].w_q.ravel()[0]
    assert s[-1] == p.expert_b2[-1]


@pytest.mark.parametrize("kw", [dict(hidden_dim=0), dict(head_dim=3), dict(max_history_len=63),
                                dict(seed=-1), dict(seed=2**64)])
def test_config_validation(kw):
    base = dict(hidden_dim=16, head_dim=4, num_blocks=2, layers_per_block=1, ffn_dim=24,
                num_tasks=3, max_history_len=64, max_candidates=32, seed=0)
    base.update(kw)
    with pytest.raises(ValueError):
        fb.ModelConfig(**base)


def test_split_sequence_mirror():
    hist = np.arange(32.0).reshape(8, 4)
    parts = fb.split_sequence(hist, 2)
    np.testing.assert_array_equal(parts[1], hist[4:])
    with pytest.raises(ValueError):
        fb.split_sequence(np.zeros((6, 2)), 4)
    with pytest.raises(NotImplementedError):
        fb.split_sequence(np.zeros((4, 2)), 2, mode="interleaved")
