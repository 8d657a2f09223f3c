"""CPU-side checks of the C ABI: libnacs.so builds for sm_100a, loads, and exports every
function include/nacs.h declares; without a GPU nacs_create fails cleanly (no fallback)."""
import os
import re
import subprocess

import pytest

from paper_1909_07673_b200 import build as nbuild
from paper_1909_07673_b200 import nacs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "nacs.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nacs_[a-z_]+)\s*\(", text)))


def test_library_builds_and_exports_header_symbols():
    path = nbuild.build()
    assert os.path.exists(path)
    declared = header_functions()
    assert len(declared) == 18, declared
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (nacs_[a-z_]+)\b", out))
    assert set(declared) <= exported, set(declared) - exported
    assert set(declared) == set(nacs.EXPORTS)
    L = nacs.lib()
    for name in declared:
        assert hasattr(L, name)


def test_sm100a_code_in_library():
    path = nbuild.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the ABI structs match the C compiler's layout of include/nacs.h."""
    import ctypes as C
    structs = {"nacs_topology": nacs.Topology, "nacs_pod_query": nacs.PodQuery,
               "nacs_requests": nacs.Requests, "nacs_placements": nacs.Placements,
               "nacs_options": nacs.Options, "nacs_stats": nacs.Stats, "nacs_graph": nacs.Graph,
               "nacs_path_query": nacs.PathQuery, "nacs_sim_config": nacs.SimConfig,
               "nacs_sim_report": nacs.SimReport}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "nacs.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = {}
    for line in subprocess.check_output([str(exe)], text=True).splitlines():
        cname, field, val = line.split()
        got[(cname, field)] = int(val)
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(nacs.NacsError):
        nacs.Context(0)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1909_07673_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src), f


def _bare_ctx():
    """A Context object without a device handle: only the binding's argument checks run."""
    c = nacs.Context.__new__(nacs.Context)
    c.device = 0
    c._h = None
    return c


def test_binding_rejects_bad_arrays():
    """tensors passed by pointer are checked for dtype, layout, device and size
    before any library call (an int64 tensor read as int32 would be garbage)."""
    import numpy as np
    import torch
    from inputs import gen
    c = _bare_ctx()
    reqs = gen.requests(3, 5)
    t = {k: (torch.from_numpy(v) if isinstance(v, np.ndarray) else v) for k, v in reqs.items()}
    with pytest.raises(ValueError, match="expected cuda:0"):
        c._requests(t)  # CPU tensors
    t64 = dict(t, cpu_min=t["cpu_min"].to(torch.int64))
    with pytest.raises(ValueError, match="dtype"):
        c._requests(t64)
    strided = dict(t, cpu_min=torch.from_numpy(np.repeat(reqs["cpu_min"], 2))[::2])
    with pytest.raises(ValueError, match="contiguous"):
        c._requests(strided)
    short = dict(reqs, cpu_min=reqs["cpu_min"][:-1])
    with pytest.raises(ValueError, match="cpu_min"):
        c._requests(short)
    with pytest.raises(ValueError, match="container_off"):
        c._requests(dict(reqs, container_off=reqs["container_off"][:-1]))
    c._requests(reqs)
    out = c._alloc_out(reqs, False)[0]
    c._check_out(out, False)
    with pytest.raises(ValueError, match="at least"):
        c._check_out(dict(out, bw_alloc=out["bw_alloc"][:-1]), False)
    with pytest.raises(ValueError, match="int32"):
        c._check_out(dict(out, status=out["status"].astype(np.int64)), False)
    with pytest.raises(ValueError, match="numpy"):
        c._check_out(dict(out, status=torch.from_numpy(out["status"])), False)
