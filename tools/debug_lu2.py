import sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle as O
import paper_1605_08771_b200 as P
ctx = P.default_context()
for n in [int(a) for a in sys.argv[1:]]:
    A = O.random_symmetric(n, n) / np.sqrt(n)
    X = O.random_block(n, 4, 1)
    for nc in (1, 4):
        for streams in (1, 4):
            ctx.set_streams(streams)
            rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.4), nc)
            res = []
            for rep in range(2):
                Y = P.apply_filter(A, rule, X)
                Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.3, 0.4), nc), X) if rep == 0 else Yo
                res.append(np.linalg.norm(Y - Yo) / np.linalg.norm(Yo))
            print(n, "nc", nc, "streams", streams, ["%.1e" % r for r in res], flush=True)
