"""Seeded random-shape sweep of the quantized path against the C oracle
(rel_err < 1e-5, the reference's own bar): rows 1..3000, columns 1..20000, k
3..8, activation rows 1..8, fp32 or fp16 activations, single calls and grouped
launches (separate or shared activations, fp16 / fp32 outputs)."""

import os

import numpy as np
import pytest

from oracle import oracle as ora

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _layer(rng, rows, cols, n_min=3, n_max=8):
    from paper_2402_10517_b200 import AnyPrecisionLayer

    codes, tables = ora.random_layer_arrays(rng, rows, cols, n_min, n_max)
    return AnyPrecisionLayer(n_min=n_min, n_max=n_max, codes=codes, centroid_tables=tables, shape=(rows, cols))


@pytest.mark.parametrize("seed", range(int(os.environ.get("APB_FUZZ_SINGLE", "12"))))
def test_random_shapes_vs_oracle(seed):
    from paper_2402_10517_b200 import engine

    rng = np.random.default_rng(1000 + seed)
    rows = int(rng.choice([1, 7, 16, 17, 100, 333, 1024, 3000]))
    cols = int(rng.choice([1, 5, 8, 1000, 1024, 1025, 4096, 5000, 11008, 20000]))
    layer = _layer(rng, rows, cols)
    prep = engine.prepare(layer)
    planes = prep.planes.cpu().numpy()
    k = int(rng.integers(3, 9))
    m = int(rng.integers(1, 9))
    fp16 = bool(rng.integers(0, 2))
    X = rng.standard_normal((m, cols)) * 10 ** rng.uniform(-2, 2)
    cfg = engine.GemvConfig(bit_width=k, activations_fp16=fp16)
    y = engine.gemm(prep, X, cfg) if m > 1 else engine.gemv(prep, X[0], cfg)[None, :]
    want = ora.gemm(planes, cols, k, layer.centroid_tables[k], ora.prep_x(X, cols, fp16), nthreads=8)
    assert y.shape == want.shape
    assert ora.rel_err(y, want) < TOL, (rows, cols, k, m, fp16, ora.rel_err(y, want))


@pytest.mark.parametrize("seed", range(int(os.environ.get("APB_FUZZ_GROUPED", "8"))))
def test_random_grouped_launches_vs_oracle(seed):
    import torch

    from paper_2402_10517_b200 import engine, plan

    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(2, 6))
    shared = bool(rng.integers(0, 2))
    cols_shared = int(rng.choice([300, 2048, 4100]))
    shapes = [(int(rng.choice([16, 50, 700, 2049])), cols_shared if shared else int(rng.choice([300, 2048, 4100])))
              for _ in range(n)]
    layers = [_layer(rng, r, c) for r, c in shapes]
    preps = [engine.prepare(L) for L in layers]
    k = int(rng.integers(3, 9))
    m = int(rng.integers(1, 9))
    y16 = bool(rng.integers(0, 2))
    p = plan.GemvPlan(preps, k, m=m, grouped=True, shared_x=shared, y_fp16=y16)
    xs = []
    for i, (r, c) in enumerate(shapes):
        if shared and i > 0:
            xs.append(xs[0])
            continue
        x = rng.standard_normal((m, c)).astype(np.float16)
        p.x[i][:, :c].copy_(torch.from_numpy(x))
        xs.append(x)
    p.run()
    torch.cuda.synchronize()
    for i, ((r, c), L, prep) in enumerate(zip(shapes, layers, preps)):
        want = ora.gemm(prep.planes.cpu().numpy(), c, k, L.centroid_tables[k],
                        ora.prep_x(xs[i].astype(np.float32), c, True), nthreads=8)
        got = p.y[i].float().cpu().numpy()
        tol = 2e-3 if y16 else TOL  # fp16 outputs: one rounding of the fp32 result
        assert ora.rel_err(got, want) < tol, (shapes, k, m, shared, y16, i, ora.rel_err(got, want))
