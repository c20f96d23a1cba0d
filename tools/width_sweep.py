"""Mantissa-width sweep (BASELINE configs[4] in 2D): measure.width_sweep.

usage: python tools/width_sweep.py [depth]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2005_03606_b200 as lzb  # noqa: E402
from paper_2005_03606_b200 import measure  # noqa: E402

if __name__ == "__main__":
    depth = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    peak = 6468.6
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    for row in measure.width_sweep(lzb.default_context(), lzb.field_sinusoid(0.9, 6.0), depth, peak):
        print(json.dumps(row))
