"""The device generator (workloads/gen_cuda.cu) reproduces workloads/gen.py bit for bit."""
import numpy as np
import pytest

from workloads import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_device_generators_match_numpy():
    from workloads import gen_cuda
    n = 100_003
    k, v = gen_cuda.u64_keys(n, lo=17)
    assert np.array_equal(k.cpu().numpy().view(np.uint64), gen.u64_keys(n, lo=17))
    assert np.array_equal(v.cpu().numpy().view(np.uint64), gen.u64_values(n, lo=17))
    q, ev, ef = gen_cuda.u64_queries(n, 50_000, lo=5, with_expect=True)
    hq, hf, hv = gen.u64_queries(n, 50_000, lo=5)
    assert np.array_equal(q.cpu().numpy().view(np.uint64), hq)
    assert np.array_equal(ef.cpu().numpy().astype(bool), hf)
    assert np.array_equal(ev.cpu().numpy().view(np.uint64), hv)
    ctx, offs = gen_cuda.string_keys(20_000, lo=3)
    hc, ho = gen.string_keys(20_000, lo=3)
    assert np.array_equal(offs.cpu().numpy().view(np.uint64), ho)
    assert np.array_equal(ctx.cpu().numpy(), hc)
    qc, qo, ids = gen_cuda.string_queries(20_000, 7_000)
    hqc, hqo, _, _ = gen.string_queries(20_000, 7_000)
    assert np.array_equal(qo.cpu().numpy().view(np.uint64), hqo)
    assert np.array_equal(qc.cpu().numpy(), hqc)


def test_device_paper_shape_strings_match_numpy():
    """The paper's Table 1 string shape (5..25 characters)."""
    from workloads import gen_cuda
    ctx, offs = gen_cuda.string_keys(30_001, lo=9, lens_range=(5, 25))
    hc, ho = gen.pack_strings(np.arange(9, 9 + 30_001, dtype=np.uint64), lens_range=(5, 25))
    lens = np.diff(ho.astype(np.int64))
    assert lens.min() == 5 and lens.max() == 25
    assert np.array_equal(offs.cpu().numpy().view(np.uint64), ho)
    assert np.array_equal(ctx.cpu().numpy(), hc)
