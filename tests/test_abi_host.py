"""C-ABI surface and host-only logic of liblzb.so (no device work).

* the library loads and exports every entry point include/lzb.h declares;
* without a GPU the context call fails loudly (no CPU fallback);
* host-side data formats (header byte, checkerboard table, geometric block)
  and the config / telemetry layer (experiment.hpp) match the reference.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from conftest import GOLDEN, ROOT
from oracle import port
from oracle import ref as refmod


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "lzb.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lzb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = lzb.lib()
    syms = declared_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_every_kernel_enters_through_pdl_wait():
    """LZB_LAUNCH may give any launch the programmatic-dependent-launch
    attribute while a cycle body is captured (engine.hpp), so every kernel's
    first statement must be lzb_pdl_enter() (griddepcontrol.wait): otherwise it
    could run before its predecessor's writes are visible."""
    src = os.path.join(ROOT, "paper_2005_03606_b200", "csrc")
    missing, count = [], 0
    for name in sorted(os.listdir(src)):
        if not name.endswith((".cu", ".cuh")):
            continue
        s = open(os.path.join(src, name)).read()
        for m in re.finditer(r"__global__", s):
            i, j = s.find("{", m.end()), s.find(";", m.end())
            if j != -1 and j < i:
                continue  # a declaration
            count += 1
            if not s[i + 1:i + 200].lstrip().startswith("lzb_pdl_enter();"):
                missing.append(f"{name}: {s[m.end():i].split('(')[0].split()[-1]}")
    assert count >= 90 and not missing, missing


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(lzb.LzbError) as e:
        lzb.Context(0)
    assert e.value.code == lzb.T.ERR_CUDA


def test_header_byte_matches_oracle_and_reference_cases():
    # test_codec.cpp:134-155
    for p1, p2, p3, cls in [(0, False, 0, 0), (5, True, 4, 1), (-1, False, 8, 2)]:
        h = lzb.pack_header(p1, p2, p3)
        assert h == port.lib().orc_pack_header(p1, int(p2), p3)
        assert lzb.unpack_header(h) == (cls, p2, p3)
    with pytest.raises(lzb.CorruptStreamError):
        lzb.unpack_header(0xC1)


def test_checkerboard_table_is_bit_identical_to_oracle():
    a = lzb.checkerboard(1, 8)
    b = port.field_from_keys({"setup": "checkerboard", "field-seed": "1", "blocks": "8"})
    assert np.array_equal(np.array(a.table[:]), np.array(b.table[:]))
    assert 1e-2 <= min(a.table[:64]) and max(a.table[:64]) <= 1e2
    for x, y in [(0.1, 0.2), (0.5, 0.5), (0.999, 0.0), (1.0, 1.0)]:
        assert lzb.lib().lzb_field_eval_host(C.byref(a), x, y) == port.lib().orc_field_eval(C.byref(b), x, y)


def test_geometric_prolongation_matches_oracle():
    assert np.array_equal(lzb.geometric_prolongation(), port.geometric())


def _keys(text):
    return lzb.config_keys(text)


def test_config_parse_and_roundtrip():
    # test_experiment.cpp:21-58
    k = _keys("# smoke experiment\nsetup = quadrant\neps-low = 1e-4   # the jump\ndepth = 3\n"
              "assembly = anarchic\ngating = off\n\n")
    assert k["setup"] == "quadrant" and float(k["eps-low"]) == 1e-4 and k["depth"] == "3"
    assert k["assembly"] == "anarchic" and k["gating"] == "off"
    text = "".join(f"{a} = {b}\n" for a, b in k.items())
    assert _keys(text) == k
    with pytest.raises(lzb.LzbError):
        _keys("nonsense-key = 1\n")
    with pytest.raises(lzb.LzbError):
        _keys("just some words\n")
    # extension keys appear only when set
    assert "schedule" not in k
    assert _keys("schedule = double\n")["schedule"] == "double"


@pytest.mark.skipif(not refmod.available(), reason="oracle/_ref not built")
def test_config_keys_match_reference_to_keys():
    buf = C.create_string_buffer(1 << 16)
    for text in ["setup = theta\ntheta = 64\nworkers = 3\n", "depth = 5\nomega = 0.6\nrhs = 1\n",
                 open(os.path.join(GOLDEN, "exp_cmp_b.cfg")).read()]:
        assert refmod.lib().ref_config_keys(text.encode(), buf, len(buf)) == 0
        want = dict(line.split(" = ", 1) for line in buf.value.decode().splitlines())
        assert _keys(text) == want


def test_emit_table_on_golden_telemetry():
    paths = [os.path.join(GOLDEN, "exp_table_t1.csv")]
    t = lzb.emit_table(paths)
    assert "theta = 1" in t and "max{n}" in t and "128.00" in t
    assert t.count("\n") == 5  # header + 4 cycles (test_experiment.cpp:132-148)
    if refmod.available():
        paths2 = paths + [os.path.join(GOLDEN, "exp_cmp_b.csv")]
        assert lzb.emit_table(paths2) == refmod.emit_table(paths2)


def test_compare_runs_on_golden_telemetry():
    a, b = os.path.join(GOLDEN, "exp_cmp_eager.csv"), os.path.join(GOLDEN, "exp_cmp_anarchic.csv")
    j = lzb.compare_runs(a, b)
    assert "cycles_to_target" in j and "final_status" in j and "converged" in j
    import json
    d = json.loads(j)
    assert d["a"]["cycles_to_target"] == 67 and d["b"]["final_status"] == "converged"
    with pytest.raises(lzb.LzbError):
        lzb.compare_runs(os.path.join(GOLDEN, "exp_cmp_a.csv"), os.path.join(GOLDEN, "exp_cmp_b.csv"))


def test_scatter_row_host():
    """scatter_row (element.cpp:39-45): the row of `corner` lands relative to
    that corner in the Stencil9 layout (dy+1)*3 + (dx+1) (types.hpp:53-58)."""
    rng = np.random.default_rng(4)
    m = rng.standard_normal(16)
    for corner in range(4):
        st = lzb.scatter_row(m, corner, np.ones(9))
        want = np.ones(9)
        for c in range(4):
            dx, dy = (c & 1) - (corner & 1), (c >> 1) - (corner >> 1)
            want[(dy + 1) * 3 + dx + 1] += m[corner * 4 + c]
        assert np.array_equal(st, want)
    with pytest.raises(lzb.LzbError):
        lzb.scatter_row(m, 4)
