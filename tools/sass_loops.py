"""Instruction mix of the backward-branch loops of one kernel in the SASS of
liblzb.so (cuobjdump -sass): used to count the DP instructions per
sub-sample of the integration kernels. Usage:
    python tools/sass_loops.py <substring of the mangled kernel name> [min_len]"""
import re
import subprocess
import sys

so = "paper_2005_03606_b200/lib/liblzb.so"
pat, min_len = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20
s = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
for p in re.split(r"\n\s+Function : ", s):
    name = p.split("\n", 1)[0]
    if pat not in name or "$" in name:
        continue
    ins = [l for l in p.split("\n") if re.search(r"/\*[0-9a-f]{4,5}\*/", l)]
    addr = lambda x: int(re.search(r"/\*([0-9a-f]{4,5})\*/", x).group(1), 16)  # noqa: E731
    print(name[-90:], len(ins), "instructions")
    for l in ins:
        m = re.search(r"\bBRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", l)
        if not m or int(m.group(1), 16) >= addr(l):
            continue
        seg = [x for x in ins if int(m.group(1), 16) <= addr(x) <= addr(l)]
        if len(seg) < min_len:
            continue
        cnt = {}
        for x in seg:
            op = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", x)
            if op:
                cnt[op.group(1)] = cnt.get(op.group(1), 0) + 1
        dp = sum(v for k, v in cnt.items() if k in ("DADD", "DMUL", "DFMA"))
        top = dict(sorted(cnt.items(), key=lambda t: -t[1])[:12])
        print(f"  loop {m.group(1)}..{hex(addr(l))}: {len(seg)} instr, DP {dp}: {top}")
