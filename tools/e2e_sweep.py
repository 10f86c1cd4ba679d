"""PCIe end-to-end sweep for the pinned-host kron_apply pipeline (cfg4).

Times the host-in/host-out matvec at several slab counts next to raw H2D,
D2H and duplex copies of the same bytes, to see how far the pipeline sits
from the box's PCIe bound.  Prints one JSON line.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_23804_b200 import operators as ops  # noqa: E402
from paper_2512_23804_b200.operators import KroneckerSumOperator, kron_apply  # noqa: E402
from paper_2512_23804_b200.problems import build_problem  # noqa: E402


def _time(fn, reps, stream):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    bundle = build_problem(4)
    op = KroneckerSumOperator(couplings=bundle.triple.matrices[: bundle.n_terms], operators=bundle.stiffness)
    x_host = np.random.default_rng(0).standard_normal((bundle.n_h, bundle.n_xi))
    xp = torch.from_numpy(x_host).pin_memory()
    wp = torch.empty_like(xp).pin_memory()
    xd = torch.empty(xp.shape, dtype=xp.dtype, device=dev)
    yd = torch.empty_like(xd)
    stream = torch.cuda.current_stream(dev)
    nbytes = xp.numel() * 8
    out = {"bytes_each_way": nbytes}
    out["h2d_ms"] = _time(lambda: xd.copy_(xp, non_blocking=True), 3, stream)
    out["d2h_ms"] = _time(lambda: wp.copy_(yd, non_blocking=True), 3, stream)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def duplex():
        s1.wait_stream(stream)
        s2.wait_stream(stream)
        with torch.cuda.stream(s1):
            xd.copy_(xp, non_blocking=True)
        with torch.cuda.stream(s2):
            wp.copy_(yd, non_blocking=True)
        stream.wait_stream(s1)
        stream.wait_stream(s2)

    out["duplex_ms"] = _time(duplex, 3, stream)
    ref = None
    for n in (8, 16, 32, 64):
        fn = lambda: ops._kron_apply_pipelined(op, xp, wp, n_slabs=n)  # noqa: E731
        ms = [_time(fn, 5, stream) for _ in range(3)]
        if ref is None:
            ref = wp.clone()
        out[f"slabs{n}_ms"] = ms
        out[f"slabs{n}_gbs"] = op.algorithmic_bytes() / (min(ms) * 1e-3) / 1e9
        out[f"slabs{n}_maxdiff"] = float((wp - ref).abs().max())
    out["public_api_ms"] = _time(lambda: kron_apply(op, xp, out=wp), 5, stream)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
