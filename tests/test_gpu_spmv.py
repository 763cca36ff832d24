"""SpMV parity on the device, through the C ABI, against the restated oracle
and the reference's own criteria (test_ellwarp.cpp:276-386, acceptance.cpp
criterion 2). The device kernels keep the reference's per-lane summation
order, so every comparison except the csr-order oracle is bitwise."""
import numpy as np
import pytest

from tests.gpu_helpers import bits, oracle_apply, rel_close, same

pytestmark = pytest.mark.gpu

KERNELS = ["csr_ref", "k1", "k1r", "k1rs", "k2", "k2r", "k2rs"]


def dev_csr(ew, m):
    return ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def test_worked_example(ew, R, golden):
    from oracle.oracle import Csr

    g = golden["worked"]
    m = Csr.make(**{k: g["matrix"][k] for k in ("nrows", "ncols")}, ro=g["matrix"]["row_offsets"],
                 ci=g["matrix"]["col_indices"], v=g["matrix"]["values"])
    a = dev_csr(ew, m)
    for kid in KERNELS:
        y = ew.Kernel(kid, a).apply(g["x"])
        assert y.tolist() == g["y"], kid
    k = ew.Kernel("k1r", a)
    fwd, inv = k.perm()
    assert fwd.tolist() == g["forward"]
    yp = k.apply_permuted(np.asarray(g["x"])[fwd])
    assert yp[inv[0]] == 121.0


@pytest.mark.parametrize("case", range(40))
def test_corpus_all_kernels(ew, R, F, case):
    m = F.random_case(case)
    x = F.random_vector(m.ncols, 5000 + case)
    oracle = R.spmv_csr(m, x)
    a = dev_csr(ew, m)
    assert np.array_equal(bits(a.spmv(x)), bits(oracle))  # csr_ref on device: bit-identical
    for ws in (4, 8, 32):
        for kid in KERNELS:
            if kid.endswith(("r", "rs")) and m.nrows != m.ncols:
                with pytest.raises(ValueError):
                    ew.Kernel(kid, a, warp_size=ws)
                continue
            y = ew.Kernel(kid, a, warp_size=ws).apply(x)
            assert np.array_equal(bits(y), bits(oracle_apply(R, kid, m, x, ws))), (kid, ws)
            assert rel_close(y, oracle, 1e-12), (kid, ws)
        if kid in ("k1", "k2"):
            pass


@pytest.mark.parametrize("case", range(0, 40, 3))
def test_corpus_k2_threshold_sweep(ew, R, F, case):
    """acceptance.cpp:168-183: the full T sweep for the K2 family."""
    m = F.random_case(case)
    x = F.random_vector(m.ncols, 6000 + case)
    oracle = R.spmv_csr(m, x)
    a = dev_csr(ew, m)
    lens = np.diff(m.row_offsets)
    lo = max(1, int(lens.min()))
    hi = max(lo, int(lens.max()))
    for ws in (4, 32):
        for t in range(lo, hi + 1, max(1, (hi - lo) // 12)):
            for kid in ("k2", "k2r", "k2rs"):
                if kid != "k2" and m.nrows != m.ncols:
                    continue
                y = ew.Kernel(kid, a, warp_size=ws, threshold=t).apply(x)
                assert np.array_equal(bits(y), bits(oracle_apply(R, kid, m, x, ws, t))), (kid, ws, t)
                assert rel_close(y, oracle, 1e-12)


def test_apply_permuted(ew, R, F):
    for case in range(0, 16):
        m = F.random_case(case)
        if m.nrows != m.ncols:
            continue
        x = F.random_vector(m.ncols, 77 + case)
        a = dev_csr(ew, m)
        for kid in ("k1r", "k1rs", "k2r", "k2rs"):
            k = ew.Kernel(kid, a, threshold=3)
            y = k.apply_permuted(x)
            assert np.array_equal(bits(y), bits(oracle_apply(R, kid, m, x, 32, 3, permuted=True))), kid
        for kid in ("csr_ref", "k1", "k2"):
            with pytest.raises(ValueError):
                ew.Kernel(kid, a).apply_permuted(x)


def test_k2_equals_k1_at_maxrow(ew, F):
    """acceptance.cpp:326-329: T >= maxrow is bitwise K1."""
    for case in range(12):
        m = F.random_case(case)
        x = F.random_vector(m.ncols, 600 + case)
        a = dev_csr(ew, m)
        t = max(1, int(np.diff(m.row_offsets).max()))
        y1 = ew.Kernel("k1", a).apply(x)
        y2 = ew.Kernel("k2", a, threshold=t).apply(x)
        assert np.array_equal(bits(y1), bits(y2))


def test_four_lane_sum(ew, golden):
    g = golden["four_lane"]["matrix"]
    a = ew.Csr(g["nrows"], g["ncols"], g["row_offsets"], g["col_indices"], g["values"])
    assert ew.Kernel("k2", a, threshold=2).apply(np.ones(8))[0] == 255.0


def test_wide_and_row_major_layouts(ew, R, F):
    """warp_size 64 (K2 through shared memory) and the row_major diagnostic."""
    m = F.powerlaw_rows(300, 1.5, 120, 3)
    x = F.random_vector(m.ncols, 17)
    a = dev_csr(ew, m)
    for t in (1, 3, 10, 40, 120):
        y = ew.Kernel("k2", a, warp_size=64, threshold=t).apply(x)
        assert np.array_equal(bits(y), bits(oracle_apply(R, "k2", m, x, 64, t)))
    lay = ew.Layout.build(a, "k1", row_major=True)
    lr = R.build_k1(m, row_major=True)
    assert np.array_equal(lay.export().values, lr.values)
    assert np.array_equal(bits(lay.spmv(x)), bits(R.spmv_layout(lr, x)))


def test_errors(ew, F):
    m = F.random_csr(5, 7, 0.5, 3)
    a = dev_csr(ew, m)
    with pytest.raises(ValueError):
        ew.Kernel("k1r", a)  # kernels.cpp:25 non-square
    with pytest.raises(ValueError):
        ew.Kernel("nope", a)
    with pytest.raises(ValueError):
        ew.Kernel("k1", a, warp_size=12)  # warp_model.cpp:8
    with pytest.raises(ValueError):
        ew.Kernel("k1", a).apply(np.ones(6))  # dimension mismatch
    with pytest.raises(ValueError):
        ew.Csr(2, 2, [0, 1, 2], [1, 0], [1.0])  # length mismatch
    with pytest.raises(ValueError):
        ew.Csr(2, 2, [0, 2, 2], [1, 0], [1.0, 1.0])  # not increasing
    with pytest.raises(ValueError):
        ew.Csr(2, 2, [0, 1, 2], [0, 2], [1.0, 1.0])  # column out of range
    with pytest.raises(ValueError):
        ew.Csr(2, 2, [0, 1, 3], [0, 1], [1.0, 1.0])  # row_offsets[n] != nnz


def test_empty_rows_and_empty_matrix(ew, R):
    from oracle.oracle import Csr

    # rows with no entries keep y = 0.0 (warp_spmv.cpp:21-24), incl. a NaN x[0]
    m = Csr.make(6, 6, [0, 0, 2, 2, 3, 3, 3], [0, 4, 5], [1.0, 2.0, 3.0])
    x = np.array([np.nan, 1, 2, 3, 4, 5], np.float64)
    a = dev_csr(ew, m)
    for kid in KERNELS:
        y = ew.Kernel(kid, a, threshold=1).apply(x)
        want = oracle_apply(R, kid, m, x, 32, 1)
        assert same(y, want), kid
    z = Csr.make(0, 0, [0], [], [])
    az = dev_csr(ew, z)
    assert ew.Kernel("k1", az).apply(np.zeros(0)).size == 0


def test_device_buffers_and_streams(ew, R, F):
    import torch

    m = F.random_case(5)
    x = F.random_vector(m.ncols, 3)
    a = dev_csr(ew, m)
    k = ew.Kernel("k1", a)
    s = torch.cuda.Stream()
    xd = torch.tensor(x, device="cuda")
    yd = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
    with torch.cuda.stream(s):
        k.apply(xd, yd, stream=s)
    s.synchronize()
    assert np.array_equal(bits(yd.cpu().numpy()), bits(oracle_apply(R, "k1", m, x)))


BASELINES = ["csr_vector", "coo", "ell", "hyb"]

# the reference's desk-scale stand-ins for the paper's 15 matrices
# (bench/fetch.cpp:16-46); config 3 runs them at Table 2 sizes in bench.py
REGISTRY = [
    "powerlaw_rows:nrows=2048,alpha=1.4,maxrow=353,seed=11",
    "powerlaw_rows:nrows=2048,alpha=0.8,maxrow=44,seed=12",
    "uniform_band:n=4096,row_len=4",
    "fem_tet_graph:n=2048,minrow=8,maxrow=81,seed=13",
    "fem_tet_graph:n=1024,minrow=2,maxrow=78,seed=14",
    "fem_tet_graph:n=1024,minrow=4,maxrow=145,seed=15",
    "fem_tet_graph:n=2048,minrow=24,maxrow=102,seed=16",
    "fem_tet_graph:n=1024,minrow=2,maxrow=81,seed=17",
    "fem_tet_graph:n=1024,minrow=18,maxrow=204,seed=18",
    "uniform_band:n=2048,row_len=39",
    "powerlaw_rows:nrows=2000,alpha=2.0,maxrow=1000,seed=19",
    "fem_tet_graph:n=2048,minrow=2,maxrow=180,seed=20",
    "fem_tet_graph:n=3129,minrow=5,maxrow=21,seed=3",
    "fem_tet_graph:n=4563,minrow=6,maxrow=22,seed=5",
    "fem_tet_graph:n=28639,minrow=6,maxrow=24,seed=30",
]


@pytest.mark.parametrize("spec", REGISTRY)
def test_paper_suite_standins_all_kernels(ew, F, spec):
    """Every kernel id on the reference's stand-ins for the paper's suite,
    bitwise against the compiled reference (K2 at three thresholds)."""
    m = F.generate(spec)
    x = F.random_vector(m.ncols, 99)
    a = dev_csr(ew, m)
    for kid in ["csr_ref", "csr_vector", "coo", "ell", "hyb", "k1", "k1r", "k1rs"]:
        assert same(ew.Kernel(kid, a).apply(x), F.apply(kid, m, x)), kid
    for t in (3, 16, 0):
        for kid in ("k2", "k2r", "k2rs"):
            assert same(ew.Kernel(kid, a, threshold=t).apply(x), F.apply(kid, m, x, threshold=t)), (kid, t)


@pytest.mark.parametrize("case", range(0, 40, 2))
def test_baseline_formats_match_reference(ew, F, case):
    """The paper's comparison formats (formats.cpp:64-235) on the device,
    bitwise against the compiled reference, every warp size the reference
    tests (acceptance.cpp criterion 2)."""
    m = F.random_case(case)
    x = F.random_vector(m.ncols, 8000 + case)
    a = dev_csr(ew, m)
    for ws in (4, 8, 32):
        for kid in BASELINES:
            y = ew.Kernel(kid, a, warp_size=ws).apply(x)
            want = F.apply(kid, m, x, warp_size=ws)
            assert same(y, want), (kid, ws)
        for k_ell in (0, 1, 3):
            y = ew.Kernel("hyb", a, warp_size=ws, hyb_k_ell=k_ell).apply(x)
            assert same(y, F.apply("hyb", m, x, warp_size=ws, hyb_k_ell=k_ell)), ("hyb", ws, k_ell)


def test_baseline_formats_long_rows_and_stored_slots(ew, F):
    """COO carries across many warp-sized chunks; stored_slots per format
    (kernels.cpp:87-99)."""
    m = F.powerlaw_rows(400, 0.9, 390, 5)
    x = F.random_vector(m.ncols, 21)
    a = dev_csr(ew, m)
    for ws in (4, 32, 64):
        for kid in BASELINES:
            k = ew.Kernel(kid, a, warp_size=ws)
            assert same(k.apply(x), F.apply(kid, m, x, warp_size=ws)), (kid, ws)
    lens = np.diff(m.row_offsets)
    assert ew.Kernel("ell", a).stored_slots == m.nrows * lens.max()
    assert ew.Kernel("coo", a).stored_slots == m.nnz
    assert ew.Kernel("csr_vector", a).stored_slots == m.nnz


def test_host_buffer_pipeline(ew, R, F):
    """ew_kernel_apply with host buffers on a large K1 (>= 2M nnz) runs as a
    staged pipeline over the kernel's own layout (x up in chunks, the warps
    in stages, finished y rows down while later stages compute): bitwise the
    device apply, also after a values-only refresh (the stage plan holds no
    values)."""
    from oracle.oracle import Csr
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.elasticity_box(30, 30, 30)
    m = Csr.make(n, n, ro, ci, v)
    assert m.nnz >= 2_000_000
    a = dev_csr(ew, m)
    k = ew.Kernel("k1", a)
    x = np.random.default_rng(5).uniform(-1.0, 1.0, n)
    import torch

    yd = k.apply(torch.tensor(x, device="cuda")).cpu().numpy()
    for _ in range(2):
        assert np.array_equal(bits(k.apply(x)), bits(yd))
    lay = R.build_k1(m)
    try:
        assert np.array_equal(bits(yd), bits(R.spmv_layout(lay, x, scatter=True)))
    finally:
        R.free(lay)
    m2 = Csr.make(n, n, ro, ci, v * 0.5 - 1.0)
    k.refresh_values(dev_csr(ew, m2))
    lay = R.build_k1(m2)
    try:
        assert np.array_equal(bits(k.apply(x)), bits(R.spmv_layout(lay, x, scatter=True)))
    finally:
        R.free(lay)


def _nan_eq(a, b):
    """Bitwise, except that any NaN equals any NaN (payloads are not part of
    the reference's semantics)."""
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(bits(a)[~na], bits(b)[~nb])


@pytest.mark.parametrize("shape", ["mesh", "random_graph"])
def test_host_buffer_pipeline_nonfinite_x0(ew, R, F, shape):
    """The reference K1 adds 0.0 * x[0] for every padding slot of a lane
    (warp_spmv.cpp:30-34), so a non-finite x[0] turns exactly the padded rows
    (and the rows that read column 0) into NaN. The host-buffer pipeline runs
    the kernel's own warps, so its y matches the reference K1 for any x:
    NaN / +-Inf at x[0], and signed zeros, on >= 2M nnz (a mesh in natural
    order, staged, and a random graph whose rows reach across all of x)."""
    import torch

    from oracle.oracle import Csr
    from paper_1501_00324_b200 import workloads as W

    if shape == "mesh":
        n, _, ro, ci, v = W.elasticity_box(30, 30, 30)
        m = Csr.make(n, n, ro, ci, v)
    else:
        m = F.fem_tet_graph(100_000, 8, 40, 7)
    assert m.nnz >= 2_000_000
    a = dev_csr(ew, m)
    k = ew.Kernel("k1", a)
    lay = R.build_k1(m)
    padded_rows = 0
    try:
        lens = np.diff(m.row_offsets)
        row_pad = np.repeat(lay.maxrows, 32)[: m.nrows] - lay.sorted_row_length
        padded_rows = int(np.count_nonzero(row_pad > 0))
        rng = np.random.default_rng(11)
        for x0 in (np.nan, np.inf, -np.inf, -0.0, 0.0):
            x = rng.uniform(-1.0, 1.0, m.ncols)
            x[1::7] = -0.0
            x[0] = x0
            want = R.spmv_layout(lay, x, scatter=True)
            yh = k.apply(x)
            yd = k.apply(torch.tensor(x, device="cuda")).cpu().numpy()
            assert _nan_eq(yh, want), x0
            assert _nan_eq(yd, want), x0
            if np.isnan(x0) or np.isinf(x0):
                # padded rows with no column-0 entry are NaN only through padding
                touches0 = np.zeros(m.nrows, bool)
                touches0[np.repeat(np.arange(m.nrows), lens)[m.col_indices == 0]] = True
                pad_only = np.zeros(m.nrows, bool)
                pad_only[lay.forward[row_pad > 0]] = True
                pad_only &= ~touches0
                assert pad_only.any() and np.isnan(yh[pad_only]).all()
    finally:
        R.free(lay)
    assert padded_rows > 0


@pytest.mark.parametrize("kid", ["k1", "k1r", "k1rs"])
def test_k1_head_split_power_law(ew, F, kid):
    """A webbase-like matrix (120k rows, one row of 4,700 entries): the
    warps of rows over 64 entries run the cooperative K1 on a side stream
    while the plain K1 runs the rest -- bitwise the reference's K1."""
    m = F.generate("powerlaw_rows:nrows=120000,alpha=1.2,maxrow=4700,seed=23")
    x = F.random_vector(m.ncols, 7)
    a = dev_csr(ew, m)
    k = ew.Kernel(kid, a)
    assert same(k.apply(x), F.apply(kid, m, x))
    x[0] = np.nan  # padding terms 0 * x[0] as the reference executes them
    assert same(k.apply(x), F.apply(kid, m, x))


def _table2_names():
    from paper_1501_00324_b200 import workloads as W

    return [t[0] for t in W.TABLE2]


@pytest.mark.parametrize("name", _table2_names())
def test_table2_size_kernels_bitwise(ew, F, name):
    """Config 3 at Table 2 sizes (the suite bench's matrices), every form
    the layouts select there -- the cooperative K1, the head split
    (webbase), 16-bit / grouped columns past 64 MB, K2 in 128-thread CTAs
    at the suite's thresholds -- bitwise the compiled reference."""
    from oracle.oracle import Csr
    from paper_1501_00324_b200 import workloads as W

    n, nc, ro, ci, v = W.table2_matrix(name)
    m = Csr.make(n, nc, ro, ci, v)
    x = F.random_vector(nc, 5)
    a = dev_csr(ew, m)
    for kid in ("k1", "k1rs"):
        assert same(ew.Kernel(kid, a).apply(x), F.apply(kid, m, x)), kid
    for t in (16, 32):
        assert same(ew.Kernel("k2", a, threshold=t).apply(x), F.apply("k2", m, x, threshold=t)), t


def _long_head_matrix(grouped):
    """Over 64 MB of slab with narrow warps (16-bit columns) and a few very
    long rows: 400k rows of 100 entries plus one of 3,000 (compact), or 150k
    nodes x 3 unknowns sharing each node's 34 columns plus one node of 3,000
    (compact + grouped)."""
    from oracle.oracle import Csr

    if grouped:
        nodes, per = 150_000, 34
        nl = np.full(nodes, per, np.int64)
        nl[5] = 3000
        n = 3 * nodes
        lens = np.repeat(nl, 3)
        node_of = np.repeat(np.arange(nodes, dtype=np.int64), 3)
    else:
        n = 400_000
        lens = np.full(n, 100, np.int64)
        lens[7] = 3000
        node_of = np.arange(n, dtype=np.int64)
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=ro[1:])
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    j = np.arange(ro[-1]) - np.repeat(ro[:-1], lens)
    cols = (np.repeat(node_of, lens) * 7 + j * 13) % n
    cols = np.sort(rows * n + cols) - rows * n
    vals = np.random.default_rng(2).uniform(0.1, 1.0, ro[-1])
    return Csr.make(n, n, ro, cols, vals)


@pytest.mark.parametrize("grouped", [False, True], ids=["compact", "grouped"])
def test_k1_head_split_compact_and_grouped(ew, F, grouped):
    """The head split on layouts over 64 MB (16-bit / grouped columns, int32
    slab dropped): the long rows' warps through k1_long_kernel reading the
    kept column form, the rest through the matching plain form -- bitwise
    the reference K1, non-finite x[0] included."""
    m = _long_head_matrix(grouped)
    a = dev_csr(ew, m)
    k = ew.Kernel("k1", a)
    i = k.info()
    assert i.narrow_slots > 0.9 * i.stored_slots
    if grouped:
        assert i.col_stream_bytes < 2 * i.stored_slots
    x = F.random_vector(m.ncols, 9)
    assert same(k.apply(x), F.apply("k1", m, x))
    x[0] = np.nan
    assert same(k.apply(x), F.apply("k1", m, x))
