import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import pytest  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_forward(name: str):
    """(config, params, history, candidates, blob) of a forward fixture."""
    import paper_2509_22681_b200 as fb

    blob = load_golden(f"forward_{name}.npz")
    dims = [int(x) for x in blob["dims"]]
    cfg = fb.ModelConfig(*dims[:8], seed=dims[8])
    params = fb.init_params(cfg)
    H, C = int(blob["H"]), int(blob["C"])
    if "history" in blob:
        hist, cand = blob["history"], blob["candidates"]
    else:
        rng = np.random.default_rng(int(blob["input_seed"]))
        hist = rng.uniform(-1.0, 1.0, (H, cfg.hidden_dim))
        cand = rng.uniform(-1.0, 1.0, (C, cfg.hidden_dim))
    return cfg, params, hist, cand, blob


FORWARD_CASES = ["cfg1", "ref_instance", "sample_json", "l2_wide", "nohist", "l3_nb4", "cfg2", "cfg3",
                 "long_hist_l2", "cfg5"]
SMALL_CASES = ["cfg1", "ref_instance", "sample_json", "l2_wide", "nohist", "l3_nb4"]


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)
