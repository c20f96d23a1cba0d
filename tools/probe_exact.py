import sys, numpy as np
sys.path.insert(0, '.')
import paper_2005_03606_b200 as lzb
from oracle import port
for text in ["setup = theta\ntheta = 16", "setup = sinusoid"]:
    t = f"{text}\ndepth = 4\nsolver = additive\nassembly = eager\nmax-cycles = 10\nomega = 0.6\nseed = 42\n"
    d = port.desc_from_keys(port.parse_keys(t))
    d.rhs = lzb.Rhs(kind=lzb.T.RHS_SINPROD, value=2 * np.pi ** 2)
    g, o = lzb.Grid(d, 42), port.Grid(d, 42)
    rg, ro = g.run(), o.run()
    print(text.split()[2], [a['residual'] == b['residual'] for a, b in zip(rg, ro)])
    print(' u exact', all(np.array_equal(g.vertices(l, 0), o.vertices(l, 0)) for l in range(5)),
          ' ops exact', all(np.array_equal(g.cells(l)['ops'], o.cells(l)['ops']) for l in range(5)),
          ' stream', g.stream_image() == o.stream_image())
