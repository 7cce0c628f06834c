"""Per-GPU filter time of one rank's node shard, measured alone on one GPU.

At G GPUs each rank factors and solves n_c/G contiguous contour nodes (the
all-reduce of Y is ~0.1 ms on NVLink and not included). This times the
filter applied with only rank 0's shard of the rule, so the strong-scaling
ceiling of a config can be read from one GPU without ranks that wait on
each other.

  python tools/shard_time.py [--config 2] [--gpus 1 2 4 8] [--steps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--factorization", default="lu", choices=["lu", "ldlt"])
    args = ap.parse_args()
    import torch

    import paper_1605_08771_b200 as P
    from paper_1605_08771_b200 import configs as CF

    c = CF.CONFIGS[args.config]
    n, nc = c.n, c.n_c
    p = c.m0 if c.m0 else 660
    lo, hi = (c.lo, c.hi) if args.config != 3 else CF.cfg3_interval()[:2]
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    A = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)
    A = (A + A.T) * (0.5 / n ** 0.5)
    ctx = P.default_context()
    ctx.set_streams(args.streams)
    ctx.set_factorization(args.factorization)
    dA = P.DeviceMatrix.from_device(A.data_ptr(), n, n, ctx)
    X = torch.randn(p, n, dtype=torch.float64, device=dev, generator=g)
    Y = torch.empty_like(X)
    rule = P.build_contour_rule(P.SearchInterval(lo, hi), nc)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    base = None
    for G in args.gpus:
        k = nc // G
        sub = P.ContourRule(rule.interval, rule.nodes[:k], rule.weights[:k])
        f = P.FilterApplier(None, sub, False, ctx=ctx, device_matrix=dA)
        for _ in range(2):
            f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if base is None:
            base = ms * G  # the first entry's shard time scaled to all n_c nodes
        flops = k * ((8.0 if args.factorization == "lu" else 4.0) / 3.0 * n ** 3 + 8.0 * n * n * p)
        print(json.dumps({"config": args.config, "factorization": args.factorization, "gpus": G, "nodes_per_gpu": k,
                          "ms_per_step": round(ms, 3), "tflops_per_gpu": round(flops / ms / 1e9, 2),
                          "speedup_vs_1": round(base / ms, 2)}),
              flush=True)
        del f


if __name__ == "__main__":
    main()
