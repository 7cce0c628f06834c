# LU/filter parity vs oracle across sizes that exercise every panel variant
import sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle as O
import paper_1605_08771_b200 as P
for n, p in [(60, 3), (130, 7), (1000, 40), (2100, 30), (4500, 20), (8300, 10)]:
    A = O.random_symmetric(n, n) / np.sqrt(n)
    X = O.random_block(n, p, 1)
    rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.4), 4)
    t0 = time.time()
    Y = P.apply_filter(A, rule, X)
    t1 = time.time()
    Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.3, 0.4), 4), X)
    print(n, p, "rel", np.linalg.norm(Y - Yo) / np.linalg.norm(Yo), "gpu s", round(t1 - t0, 3), flush=True)
