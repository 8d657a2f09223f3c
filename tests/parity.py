"""Helpers comparing the CUDA path (through the C ABI) with the CPU oracle."""
import numpy as np

from oracle import oracle as O

OUT_KEYS = ("status", "server_of_container", "cpu_alloc", "ram_alloc", "bw_alloc", "path_of_vlink")

# Per-server score tolerance (north_star): 1e-4 relative.  DESIGN.md §5 derives the FP32
# bounds (TOPSIS <= 20u, AHP <= (96 + 2 ceil(nf/32)) u relative, u = 2^-24), far inside it.
SCORE_RTOL = 1e-4


def to_np(out):
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)) for k, v in out.items()}


def assert_rank_parity(gpu, orc, label=""):
    """Mask bit-exact; best equal or inside the oracle's R14 tie set; scores within 1e-4 rel."""
    assert np.array_equal(gpu["mask"].astype(bool), orc["mask"].astype(bool)), label
    if orc["best"] < 0:
        assert gpu["best"] == -1, label
        return
    assert gpu["best"] == orc["best"] or orc["tie"][gpu["best"]], (label, gpu["best"], orc["best"])
    F = orc["mask"].astype(bool)
    g, o = gpu["scores"][F].astype(np.float64), orc["score"][F]
    err = np.abs(g - o)
    assert (err <= SCORE_RTOL * np.abs(o)).all(), (label, float(np.max(err / np.maximum(np.abs(o), 1e-300))))
    assert (gpu["scores"][~F] == 0).all(), label


def assert_schedule_parity(snap, reqs, gpu_out, method, schema, sequential, gpu_state=None, **kw):
    """Run the oracle with the GPU's servers as hints (R14 lock-step resync on excused ties)
    and require identical placements; returns the oracle counters."""
    g = to_np(gpu_out)
    orc, cnt, st = O.schedule(snap, reqs, method, schema, sequential=sequential,
                              hint=g["server_of_container"], **kw)
    assert cnt["hint_mismatch"] == 0, cnt
    for key in OUT_KEYS:
        if not np.array_equal(g[key], orc[key]):
            bad = np.nonzero(g[key] != orc[key])[0][:10]
            raise AssertionError(f"{key} differs at {bad.tolist()}: gpu {g[key][bad].tolist()} "
                                 f"oracle {orc[key][bad].tolist()} counters {cnt}")
    if gpu_state is not None:
        for key in ("cpu_res", "ram_res", "active", "link_res"):
            assert np.array_equal(np.asarray(gpu_state[key]), np.asarray(st[key])), key
    return cnt
