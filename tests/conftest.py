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


# --- BASELINE-config goldens (tests/golden/make_config_golden.py) -----------------
GOLD_FULL_VEC = 65536      # per-pixel vectors stored whole up to this length, else sampled
GOLD_VEC_SAMPLES = 32768   # seeded sample size of longer per-pixel vectors
GOLD_FULL_MAT = 256        # pose-space matrices stored whole up to this order, else by blocks
GOLD_OTHER_BLOCKS = 1500   # off-band non-zero blocks stored (seeded sample) for large matrices


def golden_vec_indices(n, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, GOLD_VEC_SAMPLES, replace=False)).astype(np.int64)


def golden_proj_vector(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


def packed_hash(P):
    """sha256 of a packed problem (pack_graph output): identifies the generated inputs."""
    import hashlib
    h = hashlib.sha256()
    for k in sorted(P):
        a = np.ascontiguousarray(np.asarray(P[k]))
        h.update(k.encode())
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def load_config_golden(cfg):
    z = np.load(os.path.join(GOLDEN_DIR, f"bcfg{cfg}.npz"), allow_pickle=False)
    out = {k: z[k] for k in z.files}
    out["meta"] = json.loads(str(out["meta"]))
    return out


def load_contract(name):
    """tests/golden/contract/<name>.npz (make_contract_golden.py): packed inputs, meta, outputs."""
    z = np.load(os.path.join(GOLDEN_DIR, "contract", name + ".npz"), allow_pickle=False)
    P = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    P["grav_G"] = float(P["grav_G"])
    P["has_Tcb"] = bool(P["has_Tcb"])
    out = {k: z[k] for k in z.files if not k.startswith("in_")}
    meta = json.loads(str(out.pop("meta")))
    meta["opts"]["frozen_keyframes"] = tuple(meta["opts"]["frozen_keyframes"])
    return P, out, meta


def config_golden_names():
    return sorted(int(os.path.basename(p)[4:-4]) for p in glob.glob(os.path.join(GOLDEN_DIR, "bcfg*.npz")))


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith("bcfg"))


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


def graph_from_packed(P, truth=None):
    """Rebuild a paper_2512_02293_b200.types FrameGraph from a packed problem dict."""
    from paper_2512_02293_b200 import types as T
    K = len(P["kid"])
    kfs = []
    for n in range(K):
        st = T.PoseState(T.Pose(T.Rotation(P["q"][n]), P["p"][n]), P["v"][n],
                         T.BiasState(P["bg"][n], P["ba"][n]), float(P["ts"][n]))
        sl = slice(P["doff"][n], P["doff"][n + 1])
        kfs.append(T.Keyframe(int(P["kid"][n]), st, P["pix"][sl], P["disp"][sl]))
    kid = P["kid"]
    edges = []
    for e in range(len(P["ei"])):
        r = slice(P["eoff"][e], P["eoff"][e + 1])
        edges.append(T.VisionEdge(int(kid[P["ei"][e]]), int(kid[P["ej"][e]]), P["epix"][r], P["tgt"][r], P["w"][r]))
    imu = []
    for f in range(len(P["fi"])):
        imu.append((int(kid[P["fi"][f]]), int(kid[P["fj"][f]]), T.PreintegratedDelta(
            float(P["f_dt"][f]), T.Rotation(P["f_dR"][f]), P["f_dp"][f], P["f_dv"][f], P["f_Jr"][f], P["f_Jp"][f],
            P["f_Jv"][f], P["f_cov"][f], T.BiasState(P["f_bhat"][f][:3], P["f_bhat"][f][3:]))))
    fx, fy, cx, cy = P["intr"]
    W = int(max(640, cx * 2 + 1))
    Hh = int(max(480, cy * 2 + 1))
    Tcb = None
    if P.get("has_Tcb", False):
        Tcb = T.Pose(T.Rotation(P["Tcb"][:4]), P["Tcb"][4:7])
    return T.FrameGraph(kfs, edges, imu, T.GravityModel(T.Rotation(P["grav_q"]), float(P["grav_G"])),
                        T.Intrinsics(fx, fy, cx, cy, W, Hh), Tcb)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


def pgba_golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "pgba", "*.npz")))


def load_pgba_golden(name):
    """tests/golden/pgba/<name>.npz (make_pgba_golden.py): packed inputs (or the stress
    generator's, regenerated and hash-checked), meta and the reference's outputs."""
    z = np.load(os.path.join(GOLDEN_DIR, "pgba", name + ".npz"), allow_pickle=False)
    out = {k: z[k] for k in z.files}
    meta = json.loads(str(out.pop("meta")))
    meta["opts"]["frozen_keyframes"] = tuple(meta["opts"]["frozen_keyframes"])
    P = {k[3:]: v for k, v in out.items() if k.startswith("in_")}
    if P:
        P["has_Tcb"] = bool(P["has_Tcb"])
        P["n_loops"] = int(P["n_loops"])
    else:
        from paper_2512_02293_b200.pgba import pack_pose_graph
        from paper_2512_02293_b200.workloads import make_pgba_workload
        P = pack_pose_graph(make_pgba_workload()[0])
        assert packed_hash(P) == meta["input_hash"], "PGBA stress generator drifted from the golden's inputs"
    return P, {k: v for k, v in out.items() if not k.startswith("in_")}, meta


def pose_graph_from_packed(P):
    """paper_2512_02293_b200.types PoseGraph from a packed pose graph (pack_pose_graph order:
    relative edges = loops without vision, then the chain)."""
    from paper_2512_02293_b200 import types as T
    K = len(P["kid"])
    kid = [int(k) for k in P["kid"]]
    S = lambda q, t, s: T.SimTransform(T.Rotation(np.array(q)), np.array(t), float(s))  # noqa: E731
    nodes = []
    for n in range(K):
        d0, d1 = int(P["doff"][n]), int(P["doff"][n + 1])
        nodes.append(T.PoseGraphNode(kid[n], S(P["sq"][n], P["st"][n], P["ss"][n]),
                                     P["pix"][d0:d1].copy() if d1 > d0 else None,
                                     P["disp"][d0:d1].copy() if d1 > d0 else None, float(P["ts"][n])))
    rel = [T.RelativePoseEdge(kid[P["ri"][r]], kid[P["rj"][r]], S(P["rq"][r], P["rt"][r], P["rs"][r]), P["rinfo"][r])
           for r in range(len(P["ri"]))]
    V = len(P["vi"])
    n_rel_loops = int(P["n_loops"]) - V
    loops = [T.LoopEdge(e.i, e.j, e) for e in rel[:n_rel_loops]]
    for v in range(V):
        i, j = kid[P["vi"][v]], kid[P["vj"][v]]
        r0, r1 = int(P["veoff"][v]), int(P["veoff"][v + 1])
        vis = T.VisionEdge(i, j, P["vpix"][r0:r1], P["vtgt"][r0:r1], P["vw"][r0:r1])
        loops.append(T.LoopEdge(i, j, T.RelativePoseEdge(i, j, T.SimTransform.identity(), np.eye(7)), vis))
    fx, fy, cx, cy = P["intr"]
    intr = T.Intrinsics(fx, fy, cx, cy, int(max(640, 2 * cx + 1)), int(max(480, 2 * cy + 1))) if V else None
    Tcb = T.Pose(T.Rotation(P["Tcb"][:4]), P["Tcb"][4:7]) if bool(P["has_Tcb"]) else None
    gap = min([lp.j - lp.i for lp in loops] + [55])
    return T.PoseGraph(nodes, rel[n_rel_loops:], loops, intr, Tcb, min_loop_gap=gap)


def init_golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "init", "*.npz")))


def load_init_golden(name):
    z = np.load(os.path.join(GOLDEN_DIR, "init", name + ".npz"), allow_pickle=False)
    P = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    P["grav_G"] = float(P["grav_G"])
    P["has_Tcb"] = bool(P["has_Tcb"])
    out = {k: z[k] for k in z.files if not k.startswith("in_")}
    out["meta"] = json.loads(str(out["meta"]))
    return P, out
