"""Regenerate the golden telemetry fixtures from the UNMODIFIED reference.

Runs the reference's own run_experiment (oracle/_ref, compiled in place from
/root/reference/proj/src by oracle/Makefile) on the exact configurations of
the reference tests that produced proj/exp_*.csv (test_experiment.cpp:11-17,
21-158) and writes the CSVs here. They are byte-identical to the files
committed in the reference tree (checked below when that tree is present).

Usage: python tests/golden/make_golden.py
"""
import filecmp
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

SMOKE = "setup = constant\ndepth = 2\nmax-cycles = 300\ntiming = off\n"
CASES = {
    "exp_smoke.csv": SMOKE,
    "exp_cmp_eager.csv": SMOKE + "assembly = eager\n",
    "exp_cmp_anarchic.csv": SMOKE + "assembly = anarchic\n",
    "exp_cmp_a.csv": SMOKE,
    "exp_cmp_b.csv": SMOKE + "setup = theta\ntheta = 16\nmax-cycles = 5\n",
    "exp_table_t1.csv": "setup = theta\ntheta = 1\ndepth = 2\nmax-cycles = 4\ntiming = off\n",
}


def main():
    for name, text in CASES.items():
        out = os.path.join(HERE, name)
        ref.run_experiment_text(text + f"csv = {out}\n")
        with open(os.path.join(HERE, name.replace(".csv", ".cfg")), "w") as f:
            f.write(text)
        theirs = os.path.join("/root/reference/proj", name)
        same = filecmp.cmp(out, theirs, shallow=False) if os.path.exists(theirs) else None
        print(name, "identical to reference tree" if same else ("reference tree absent" if same is None else "DIFFERS"))


if __name__ == "__main__":
    main()
