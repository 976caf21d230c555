import glob
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device and the built libvba")


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)
    P = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    for k in ("grav_G",):
        P[k] = float(P[k])
    P["has_Tcb"] = bool(P["has_Tcb"])
    out = {k[4:]: z[k] for k in z.files if k.startswith("out_")}
    out["report"] = json.loads(str(out["report"]))
    opts = json.loads(str(z["opts"]))
    opts["frozen_keyframes"] = tuple(opts["frozen_keyframes"])
    return P, out, opts


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
