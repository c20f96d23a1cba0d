"""Every kernel launched through LZB_LAUNCH may carry the programmatic
dependent launch attribute (engine.hpp: PdlScope), so every __global__
function must wait on its predecessor first: its body starts with
lzb_pdl_enter() (nothing enforced this). A source check, no GPU."""
import glob
import os
import re

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2005_03606_b200", "csrc")


def _kernel_bodies(src):
    for m in re.finditer(r"__global__\s+void\s+(?:__launch_bounds__\([^)]*\)\s*)?(\w+)\s*\(", src):
        depth, j = 1, m.end()
        while depth:
            depth += {"(": 1, ")": -1}.get(src[j], 0)
            j += 1
        rest = src[j:].lstrip()
        if rest.startswith(";"):  # a declaration
            continue
        assert rest.startswith("{"), m.group(1)
        yield m.group(1), rest[1:].lstrip()


def test_every_kernel_enters_through_lzb_pdl_enter():
    files = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")))
    seen, missing = 0, []
    for f in files:
        for name, body in _kernel_bodies(open(f).read()):
            seen += 1
            if not body.startswith("lzb_pdl_enter();"):
                missing.append(f"{os.path.basename(f)}:{name}")
    assert seen >= 120, seen  # the scan found the kernels at all
    assert not missing, missing
