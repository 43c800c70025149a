"""GPU parity: libkkspgemm.so (sm_100a kernels, called through the C ABI)
against the oracle and the reference's golden output.

The contract (BASELINE.json north_star): C's row offsets and per-row sorted
columns bit-exact, fp64 values within 1e-12 relative.  The kernels preserve the
reference's first-touch column order and left-to-right summation order, so the
tests below demand the stronger property — raw columns and value bits identical
to the reference — and check the contractual one as well.
"""
import hashlib

import numpy as np
import pytest

from conftest import csr_from_triplets, load_instances, random_csr

pytestmark = pytest.mark.gpu

TOL = 1e-12  # north_star: fp64 relative tolerance per entry


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def kk():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1801_03065_b200 as kk
    kk.lib()  # fails loudly when the extension is missing
    return kk


def run(kk, a, b, cfg=None):
    res = kk.multiply(a, b, cfg)
    c = res.c.to_host()
    return res, c


def assert_parity(oracle, a, b, c, exact=True):
    ro = oracle.symbolic_row_offsets(a, b)
    assert np.array_equal(c.row_offsets, ro), "row offsets differ"
    cols, vals = oracle.numeric(a, b, ro)
    # contractual: per-row sorted columns identical, values within 1e-12
    sc, sv = oracle.sort_rows(ro, cols, vals)
    gc, gv = oracle.sort_rows(ro, c.col_indices, c.values)
    assert np.array_equal(sc, gc), "sorted columns differ"
    assert oracle.max_rel_error(sv, gv) <= TOL
    if exact:  # stronger: the reference's raw order and value bits
        assert np.array_equal(c.col_indices, cols), "first-touch column order differs"
        assert np.array_equal(c.values.view(np.int64), vals.view(np.int64)), "value bits differ"


def test_hand_3x3(kk, oracle, kats):
    k = kats["hand_3x3"]
    a = csr_from_triplets(3, 3, k["a"])
    b = csr_from_triplets(3, 3, k["b"])
    for acc in (kk.AccumulatorKind.LL, kk.AccumulatorKind.LP, kk.AccumulatorKind.Dense):
        cfg = kk.SpgemmConfig(accumulator=acc)
        h = kk.symbolic(a, b, cfg)
        assert h.c_row_offsets.tolist() == [0, 3, 4, 7]
        assert h.nnz_c() == 7
        c = kk.numeric(a, b, h).to_host()
        assert c.col_indices.tolist() == k["reference_raw_cols"]
        assert c.values.tolist() == k["reference_raw_vals"]


def test_identity_and_empty_rows(kk, oracle):
    eye = csr_from_triplets(10, 10, [(i, i, 1.0) for i in range(10)])
    h = kk.symbolic(eye, eye)
    assert h.c_row_offsets.tolist() == list(range(11))
    assert h.max_row_size == 1
    a = csr_from_triplets(3, 2, [(1, 0, 2.0)])
    b = csr_from_triplets(2, 2, [(0, 1, 4.0)])
    _, c = run(kk, a, b)
    assert c.row_offsets.tolist() == [0, 0, 1, 1]
    assert c.values.tolist() == [8.0]


def test_cancellation_kept(kk, kats):
    k = kats["cancellation"]
    a = csr_from_triplets(*k["a_shape"], k["a"])
    b = csr_from_triplets(*k["b_shape"], k["b"])
    _, c = run(kk, a, b)
    assert c.nnz() == 1 and c.values.tolist() == [0.0]


def test_flops_and_compression_report(kk, oracle, kats):
    k = kats["flops_5_0"]
    a = csr_from_triplets(*k["a_shape"], k["a"])
    b = csr_from_triplets(*k["b_shape"], k["b"])
    h = kk.symbolic(a, b)
    assert h.per_row_flops().tolist() == [5, 0]
    assert h.flops.total_flops == 5 and h.flops.max_row_flops == 5
    for name in ("gate_exact_15", "gate_16_of_20"):
        g = kats[name]
        b = csr_from_triplets(1, g["k"], [(0, c, 1.0) for c in g["b_cols"]])
        a = csr_from_triplets(1, 1, [(0, 0, 1.0)])
        h = kk.symbolic(a, b)
        assert h.compression.compressed_flops == g["compressed_flops"]
        assert h.compression.applied == g["applied"]


def test_golden_instances(kk, oracle):
    """The reference's own outputs (tests/golden/instances.npz), bit for bit."""
    for inst in load_instances():
        a, b = inst["a"], inst["b"]
        res, c = run(kk, a, b)
        h = res.handle
        assert np.array_equal(h.per_row_flops(), inst["per_row_flops"])
        assert h.flops.total_flops == inst["meta"]["total_flops"]
        assert h.compression.compressed_flops == inst["meta"]["compressed_flops"]
        assert h.compression.applied == bool(inst["meta"]["applied"])
        assert h.max_row_size == inst["meta"]["max_row_size"]
        assert h.symbolic_choice.accumulator == inst["meta"]["sym_acc"]
        assert h.symbolic_choice.effective_k == inst["meta"]["sym_effk"]
        assert h.numeric_choice.accumulator == inst["meta"]["num_acc"]
        assert h.numeric_choice.l2_capacity == inst["meta"]["num_l2"]
        assert np.array_equal(c.row_offsets, inst["c_ro"])
        assert np.array_equal(c.col_indices, inst["c_ci"])
        assert np.array_equal(c.values.view(np.int64), inst["c_v"].view(np.int64))


@pytest.mark.parametrize("acc", [1, 2, 3])
@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("l1", [0, 1, 40])
def test_every_accumulator_scheme_and_level(kk, oracle, acc, scheme, l1):
    """engine_test.cpp:76-135 / acceptance c1, c3: every accumulator x scheme,
    with the level-1 table forced tiny so rows escalate to the HBM pool."""
    if acc == 3 and l1 == 40:
        pytest.skip("dense is single-level")
    rng = np.random.default_rng(1000 * acc + 10 * scheme + l1)
    allocs = 0
    for it in range(6):
        m, n, k = (int(x) for x in rng.integers(1, 150, 3))
        a = random_csr(rng, m, n, 0.1, shuffle=bool(it % 2))
        b = random_csr(rng, n, k, 0.1, shuffle=bool(it % 2))
        cfg = kk.SpgemmConfig(accumulator=acc, scheme=scheme, l1_capacity=l1)
        h = kk.symbolic(a, b, cfg)
        st = kk.PhaseStats()
        c = kk.numeric(a, b, h, st).to_host()
        assert_parity(oracle, a, b, c)
        allocs += h.symbolic_stats.pool_allocations + st.pool_allocations
    if l1 == 1 and acc != 3:
        assert allocs >= 1  # engine_test.cpp:118-119


@pytest.mark.parametrize("acc", [0, 1, 2])
@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("l1", [1, 7, 40])
def test_phase_stats_match_reference(kk, reference, acc, scheme, l1):
    """PhaseStats carry the reference's meaning (engine.cpp:78-87,
    memory_pool.cpp allocation_count): pool_allocations = rows whose distinct
    keys overflow the level-1 accumulator, l2_inserts = products of keys past
    its capacity.  Equal to the reference's own counters, both phases."""
    rng = np.random.default_rng(500 + 100 * acc + 10 * scheme + l1)
    for it in range(3):
        m, n, k = (int(x) for x in rng.integers(20, 160, 3))
        a = random_csr(rng, m, n, 0.12, shuffle=bool(it % 2))
        b = random_csr(rng, n, k, 0.12, shuffle=bool(it % 2))
        cfg = kk.SpgemmConfig(accumulator=acc, scheme=scheme, l1_capacity=l1)
        h = kk.symbolic(a, b, cfg)
        st = kk.PhaseStats()
        kk.numeric(a, b, h, st)
        rh = reference.symbolic(a, b, accumulator=acc, scheme=scheme, l1_capacity=l1)
        info = rh.info()
        _, _, rst = rh.numeric()
        assert h.symbolic_stats.pool_allocations == info["sym_pool_allocations"]
        assert h.symbolic_stats.l2_inserts == info["sym_l2_inserts"]
        assert st.pool_allocations == rst["pool_allocations"]
        assert st.l2_inserts == rst["l2_inserts"]


@pytest.mark.parametrize("acc", [1, 2])
def test_pool_many2many_budget_halving(kk, oracle, reference, acc):
    """plan_pool (memory_pool.cpp:83-109): many2many chunk claims with a budget
    that halves the chunk count to a handful; results stay bit-exact and the
    statistics equal the reference's under the same budget."""
    rng = np.random.default_rng(71 + acc)
    a = random_csr(rng, 300, 200, 0.1)
    b = random_csr(rng, 200, 250, 0.1)
    probe = kk.symbolic(a, b, kk.SpgemmConfig(accumulator=acc, l1_capacity=1))
    bound = max(probe.numeric_choice.l2_capacity, probe.symbolic_choice.l2_capacity)
    budget = 3 * ((bound + 1) // 2 * 2 * 32)  # three reference chunks
    for mode in (kk.PoolMode.Many2Many, kk.PoolMode.One2One):
        cfg = kk.SpgemmConfig(accumulator=acc, l1_capacity=1, pool_mode=mode, pool_budget_bytes=budget)
        h = kk.symbolic(a, b, cfg)
        st = kk.PhaseStats()
        c = kk.numeric(a, b, h, st).to_host()
        assert_parity(oracle, a, b, c)
        rh = reference.symbolic(a, b, accumulator=acc, l1_capacity=1, pool_mode=mode, pool_budget_bytes=budget)
        _, _, rst = rh.numeric()
        assert st.pool_allocations == rst["pool_allocations"] > 0
        assert st.l2_inserts == rst["l2_inserts"] > 0


def test_pool_budget_below_one_chunk(kk, reference):
    """PoolSizingError when one chunk exceeds the budget (memory_pool.cpp:97-99),
    raised by the phase whose resolved accumulator is LL/LP, as the reference does."""
    rng = np.random.default_rng(73)
    a = random_csr(rng, 60, 60, 0.2)
    b = random_csr(rng, 60, 60, 0.2)
    for acc in (1, 2):
        with pytest.raises(kk.PoolSizingError):
            kk.symbolic(a, b, kk.SpgemmConfig(accumulator=acc, pool_budget_bytes=16))
        with pytest.raises(RuntimeError, match="exceeds the memory budget"):
            reference.symbolic(a, b, accumulator=acc, pool_budget_bytes=16)
    # Dense (Auto on a small domain) is single-level: no pool, no error
    h = kk.symbolic(a, b, kk.SpgemmConfig(pool_budget_bytes=16))
    assert h.symbolic_choice.accumulator == kk.AccumulatorKind.Dense
    reference.symbolic(a, b, pool_budget_bytes=16)
    # numeric raises when only its own choice needs a pool
    h2 = kk.symbolic(a, b)
    h2.set_numeric(kk.SpgemmConfig(pool_budget_bytes=16),
                   kk.ResolvedConfig(accumulator=kk.AccumulatorKind.LL, scheme=0, l1_capacity=4,
                                     effective_k=60, l2_capacity=60))
    with pytest.raises(kk.PoolSizingError):
        kk.numeric(a, b, h2, kk.PhaseStats())


def test_ample_l1_never_touches_pool(kk):
    rng = np.random.default_rng(67)
    a = random_csr(rng, 50, 50, 0.1)
    b = random_csr(rng, 50, 50, 0.1)
    h = kk.symbolic(a, b, kk.SpgemmConfig(accumulator=kk.AccumulatorKind.LL))
    st = kk.PhaseStats()
    kk.numeric(a, b, h, st)
    assert h.symbolic_stats.pool_allocations == 0 and st.pool_allocations == 0


def test_compression_modes_agree(kk, oracle):
    """engine_test.cpp:191-202 / acceptance c5."""
    rng = np.random.default_rng(79)
    for it in range(8):
        a = random_csr(rng, 150, 150, 0.04 + 0.02 * (it % 3), shuffle=bool(it % 2))
        b = random_csr(rng, 150, 150, 0.04, shuffle=bool(it % 2))
        on = kk.symbolic(a, b, kk.SpgemmConfig(compression=kk.CompressionMode.Always))
        off = kk.symbolic(a, b, kk.SpgemmConfig(compression=kk.CompressionMode.Never))
        assert on.compression.applied and not off.compression.applied
        assert np.array_equal(on.c_row_offsets, off.c_row_offsets)
        assert np.array_equal(on.c_row_offsets, oracle.symbolic_row_offsets(a, b))


def test_reuse_exact_and_linear(kk):
    """engine_test.cpp:204-224: numeric(2A) == multiply(2A) bitwise, and 2x linearity."""
    rng = np.random.default_rng(83)
    a = random_csr(rng, 60, 60, 0.1)
    b = random_csr(rng, 60, 60, 0.1)
    h = kk.symbolic(a, b)
    a2 = kk.CsrMatrix(a.num_rows, a.num_cols, a.row_offsets, a.col_indices, a.values * 2.0, True)
    c_reuse = kk.numeric(a2, b, h).to_host()
    c_fresh = kk.multiply(a2, b).c.to_host()
    assert np.array_equal(c_reuse.col_indices, c_fresh.col_indices)
    assert np.array_equal(c_reuse.values.view(np.int64), c_fresh.values.view(np.int64))
    c_base = kk.numeric(a, b, h).to_host()
    assert np.array_equal(c_reuse.values, 2.0 * c_base.values)


def test_reuse_rejects_mismatch(kk):
    rng = np.random.default_rng(89)
    a = random_csr(rng, 30, 30, 0.2)
    b = random_csr(rng, 30, 30, 0.2)
    h = kk.symbolic(a, b)
    wrong = random_csr(rng, 31, 30, 0.2)
    with pytest.raises(kk.ReuseError):
        kk.numeric(wrong, b, h)
    trimmed = kk.CsrMatrix(a.num_rows, a.num_cols, a.row_offsets.copy(), a.col_indices, a.values, True)
    trimmed.row_offsets[-1] -= 1
    with pytest.raises(kk.ReuseError):
        kk.numeric(trimmed, b, h)


def test_structure_mismatch_is_reported_not_hung(kk):
    """Same dimensions and nnz but a different B structure: the reference throws
    logic_error (engine.cpp:238-245); the kernels must report it, never spin."""
    rng = np.random.default_rng(11)
    for flat in (False, True):
        n = 40 if not flat else 400
        a = random_csr(rng, 30, n, 0.3 if not flat else 0.02)
        b = random_csr(rng, n, 50, 0.2)
        h = kk.symbolic(a, b)
        # move every entry of B to column 0..: same nnz, far fewer distinct columns
        b2 = kk.CsrMatrix(b.num_rows, b.num_cols, b.row_offsets, b.col_indices.copy(), b.values, False)
        for i in range(b2.num_rows):
            lo, hi = b2.row_offsets[i], b2.row_offsets[i + 1]
            b2.col_indices[lo:hi] = (np.arange(hi - lo) * 7 + i) % b2.num_cols
        with pytest.raises(kk.InternalError):
            kk.numeric(a, b2, h, kk.PhaseStats())


def _scaled(kk, x, f):
    return kk.CsrMatrix(x.num_rows, x.num_cols, x.row_offsets, x.col_indices, x.values * f, x.sorted_rows)


@pytest.mark.parametrize("shape", [(300, 300, 300, 0.08), (120, 2000, 400, 0.03)])
@pytest.mark.parametrize("sort", [False, True])
def test_replay_passes_bitwise(kk, oracle, shape, sort):
    """Structure reuse (engine.hpp:42-56): pass 2 records the slot map, passes
    3+ replay it (kk_replay.cu); every pass must equal a fresh multiply bit
    for bit.  Shapes give 1-byte (rows <= 256) and 2-byte slots."""
    m, n, k, d = shape
    rng = np.random.default_rng(int(1e6 * d) + m)
    a = random_csr(rng, m, n, d, shuffle=True)
    b = random_csr(rng, n, k, d * 3 if n > 1000 else d, shuffle=True)
    cfg = kk.SpgemmConfig(sort_output=sort)
    h = kk.symbolic(a, b, cfg)
    assert h.replay_state == 1, "Thread-Sequential plan with warp-table rows must be replay-eligible"
    if m == 120:
        assert h.max_row_size > 256
    for p in range(6):
        ap, bp = _scaled(kk, a, 1.0 + 0.125 * p), _scaled(kk, b, 1.0 - 0.0625 * p)
        st = kk.PhaseStats()
        c = kk.numeric(ap, bp, h, st).to_host()
        assert h.replay_state == (1 if p == 0 else 2)
        fresh = kk.multiply(ap, bp, cfg).c.to_host()
        assert np.array_equal(c.row_offsets, fresh.row_offsets)
        assert np.array_equal(c.col_indices, fresh.col_indices)
        assert np.array_equal(c.values.view(np.int64), fresh.values.view(np.int64))
        if not sort:
            assert_parity(oracle, ap, bp, c)


def test_replay_falls_back_on_structure_change(kk, oracle):
    rng = np.random.default_rng(23)
    a = random_csr(rng, 200, 200, 0.1)
    b = random_csr(rng, 200, 200, 0.1)
    h = kk.symbolic(a, b)
    for _ in range(3):
        kk.numeric(a, b, h)
    assert h.replay_state == 2
    # same nnz, same row lengths, permuted columns inside B's rows: C's
    # structure (and first-touch order) changes, so the map must not be used
    b2 = kk.CsrMatrix(b.num_rows, b.num_cols, b.row_offsets, b.col_indices.copy(), b.values, False)
    for i in range(b2.num_rows):
        lo, hi = b2.row_offsets[i], b2.row_offsets[i + 1]
        b2.col_indices[lo:hi] = b2.col_indices[lo:hi][::-1]
    c2 = kk.numeric(a, b2, h, kk.PhaseStats()).to_host()  # same column sets: a valid reuse
    assert_parity(oracle, a, b2, c2)
    c = kk.numeric(a, b, h).to_host()
    assert_parity(oracle, a, b, c)
    # same nnz, different column sets: the hashing kernels report the mismatch
    b3 = kk.CsrMatrix(b.num_rows, b.num_cols, b.row_offsets, b.col_indices.copy(), b.values, False)
    for i in range(b3.num_rows):
        lo, hi = b3.row_offsets[i], b3.row_offsets[i + 1]
        b3.col_indices[lo:hi] = np.arange(hi - lo) % b3.num_cols
    with pytest.raises(kk.InternalError):
        kk.numeric(a, b3, h, kk.PhaseStats())


def test_replay_detects_compensating_swaps(kk, oracle):
    """Edits that keep two moments of B's column array (adjacent swaps with
    opposite gaps in two rows, and a (+1,-2,+1) change at three consecutive
    positions) change C's first-touch order: the recorded slot map must not be
    replayed for them (kk_replay.cu fingerprint)."""
    rng = np.random.default_rng(31)
    n, k = 64, 200  # B rows of ~15 entries: the Thread-Sequential (replayable) plan
    rows = []
    for i in range(n):
        pool = [c for c in range(k) if c not in (3, 4, 7, 8, 20, 21, 22)]
        rows.append(list(rng.choice(pool, size=13, replace=False)))
    rows[5] = [3, 4] + rows[5]      # ascending pair, gap 1
    rows[40] = [8, 7] + rows[40]    # descending pair, gap 1
    rows[17] = [20, 22, 21] + rows[17][:10]
    ro = np.zeros(n + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=ro[1:])
    b = kk.CsrMatrix(n, k, ro, np.concatenate(rows).astype(np.int32), rng.uniform(-1, 1, int(ro[-1])), False)
    a = random_csr(rng, 80, n, 0.3)
    h = kk.symbolic(a, b)
    for _ in range(3):
        kk.numeric(a, b, h)
    assert h.replay_state == 2
    edits = []
    b2 = b.col_indices.copy()
    b2[ro[5]:ro[5] + 2] = [4, 3]
    b2[ro[40]:ro[40] + 2] = [7, 8]
    edits.append(b2)
    b3 = b.col_indices.copy()
    b3[ro[17]:ro[17] + 3] = [21, 20, 22]  # deltas (+1, -2, +1)
    edits.append(b3)
    for cols in edits:
        bx = kk.CsrMatrix(n, k, ro, cols, b.values, False)
        c = kk.numeric(a, bx, h, kk.PhaseStats()).to_host()
        assert_parity(oracle, a, bx, c)
    c = kk.numeric(a, b, h).to_host()
    assert_parity(oracle, a, b, c)


def test_row_block_errors_survive_later_blocks(kk):
    """A device error raised by one row block of a pass stays visible until
    the pass is checked (host.multiply_host calls check after its last block):
    later blocks must not clear it."""
    import torch
    rng = np.random.default_rng(37)
    a = random_csr(rng, 200, 200, 0.1)
    b = random_csr(rng, 200, 200, 0.1)
    h = kk.symbolic(a, b)
    bad = kk.CsrMatrix(b.num_rows, b.num_cols, b.row_offsets, b.col_indices.copy(), b.values, False)
    for i in range(bad.num_rows):
        lo, hi = bad.row_offsets[i], bad.row_offsets[i + 1]
        bad.col_indices[lo:hi] = np.arange(hi - lo) % bad.num_cols
    nnz = h.nnz_c()
    cols = torch.empty(nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
    kk.numeric_rows(a, bad, h, 0, 100, cols, vals)   # block 0: structure mismatch
    kk.numeric_rows(a, b, h, 100, 200, cols, vals)   # block 1: clean
    with pytest.raises(kk.InternalError):
        h.check()
    kk.numeric_rows(a, b, h, 0, 100, cols, vals)     # a new pass starts at row 0
    kk.numeric_rows(a, b, h, 100, 200, cols, vals)
    h.check()


def test_products_in_a_structurally_empty_row_are_reported(kk):
    """A reused handle whose new A puts products into a row of C the symbolic
    pass left empty raises (NumericSink::finish, engine.cpp:238-239) instead
    of dropping them: same nnz, one entry moved from a B row that is empty to
    one that is not, into an empty A row."""
    rng = np.random.default_rng(41)
    trips_b = [(i, int(c), float(rng.uniform(-1, 1))) for i in range(40) if i != 7
               for c in rng.choice(50, 6, replace=False)]
    b = csr_from_triplets(40, 50, trips_b)
    base = [(r, int(c), 1.0) for r in (0, 1, 2, 4, 6, 8, 9) for c in rng.choice(40, 4, replace=False) if c != 7]
    a = csr_from_triplets(10, 40, base + [(5, 7, 2.0), (5, 12, 3.0)])
    a2 = csr_from_triplets(10, 40, base + [(3, 20, 2.0), (5, 12, 3.0)])
    assert a.nnz() == a2.nnz()
    h = kk.symbolic(a, b)
    assert h.c_row_offsets[4] == h.c_row_offsets[3]  # row 3 of C is empty
    kk.numeric(a, b, h, kk.PhaseStats())
    with pytest.raises(kk.InternalError):
        kk.numeric(a2, b, h, kk.PhaseStats())


def test_replay_row_block_views(kk, oracle):
    rng = np.random.default_rng(29)
    a = random_csr(rng, 400, 150, 0.12)
    b = random_csr(rng, 150, 160, 0.12)
    da, db = a.to_device(), b.to_device()
    ro = oracle.symbolic_row_offsets(a, b)
    full_cols, full_vals = oracle.numeric(a, b, ro)
    lo, hi = 133, 311
    blk = da.row_block(lo, hi)
    h = kk.symbolic(blk, db)
    for _ in range(4):
        c = kk.numeric(blk, db, h).to_host()
        assert np.array_equal(c.col_indices, full_cols[ro[lo]:ro[hi]])
        assert np.array_equal(c.values.view(np.int64), full_vals[ro[lo]:ro[hi]].view(np.int64))
    assert h.replay_state == 2


def test_contract_errors(kk):
    a = csr_from_triplets(2, 3, [])
    b = csr_from_triplets(2, 2, [])
    with pytest.raises(kk.ContractError):
        kk.symbolic(a, b)


def test_sort_output(kk, oracle):
    rng = np.random.default_rng(97)
    a = random_csr(rng, 50, 50, 0.15)
    b = random_csr(rng, 50, 50, 0.15)
    c = kk.multiply(a, b, kk.SpgemmConfig(sort_output=True)).c.to_host()
    assert c.sorted_rows
    for i in range(c.num_rows):
        seg = c.col_indices[c.row_offsets[i]:c.row_offsets[i + 1]]
        assert np.all(np.diff(seg) > 0)
    ro = oracle.symbolic_row_offsets(a, b)
    sc, sv = oracle.sort_rows(ro, *oracle.numeric(a, b, ro))
    assert np.array_equal(sc, c.col_indices)
    assert np.array_equal(sv.view(np.int64), c.values.view(np.int64))


def test_row_block_views(kk, oracle):
    """Row shards (multi-GPU partitions) are row-offset views of one matrix."""
    rng = np.random.default_rng(5)
    a = random_csr(rng, 200, 120, 0.08)
    b = random_csr(rng, 120, 90, 0.1)
    da, db = a.to_device(), b.to_device()
    ro = oracle.symbolic_row_offsets(a, b)
    full_cols, full_vals = oracle.numeric(a, b, ro)
    for lo, hi in ((0, 77), (77, 150), (150, 200)):
        res = kk.multiply(da.row_block(lo, hi), db)
        c = res.c.to_host()
        assert np.array_equal(c.row_offsets, ro[lo:hi + 1] - ro[lo])
        assert np.array_equal(c.col_indices, full_cols[ro[lo]:ro[hi]])
        assert np.array_equal(c.values.view(np.int64), full_vals[ro[lo]:ro[hi]].view(np.int64))


def test_triple_product(kk, oracle):
    """engine_test.cpp:266-280: R*(A*P) with R = P^T, AP fed back unsorted."""
    from paper_1801_03065_b200 import generators as G
    a = G.laplace3d(10)
    p = G.aggregation(10)
    r = G.transpose(p)
    ap = kk.multiply(a, p)
    rap = kk.multiply(r, ap.c).c.to_host()
    ro1 = oracle.symbolic_row_offsets(a, p)
    apc, apv = oracle.numeric(a, p, ro1)
    ap_host = kk.CsrMatrix(a.num_rows, p.num_cols, ro1, apc, apv, False)
    assert_parity(oracle, r, ap_host, rap)


CONFIG_CASES = ["c1_2d_n100", "c2_3d_n16", "c3_ap_n12", "c4_rmat_s10", "c5_3d_n20"]


@pytest.mark.parametrize("name", CONFIG_CASES)
def test_configs_reduced_vs_reference_digests(kk, config_golden, name):
    """BASELINE configs at reduced scale: the reference's raw output digests."""
    from paper_1801_03065_b200 import generators as G
    make = {"c1_2d_n100": lambda: (G.laplace2d(100), None), "c2_3d_n16": lambda: (G.laplace3d(16), None),
            "c3_ap_n12": lambda: (G.laplace3d(12), G.aggregation(12)),
            "c4_rmat_s10": lambda: (G.rmat(10, 16, 1), None), "c5_3d_n20": lambda: (G.laplace3d(20), None)}
    a, b = make[name]()
    b = a if b is None else b
    g = config_golden[name]
    res, c = run(kk, a, b)
    h = res.handle
    assert h.flops.total_flops == g["total_flops"]
    assert h.compression.compressed_flops == g["compressed_flops"]
    assert h.symbolic_choice.accumulator == g["sym_acc"]
    assert digest(c.row_offsets) == g["row_offsets_sha256"]
    assert digest(c.col_indices) == g["raw_cols_sha256"]
    assert digest(c.values) == g["raw_vals_sha256"]
    if name == "c3_ap_n12":
        r = G.transpose(b)
        rap = kk.multiply(r, res.c).c.to_host()
        g2 = config_golden["c3_rap_n12"]
        assert digest(rap.row_offsets) == g2["row_offsets_sha256"]
        assert digest(rap.col_indices) == g2["raw_cols_sha256"]
        assert digest(rap.values) == g2["raw_vals_sha256"]


def test_c1_full_size_vs_oracle(kk, oracle):
    """Config 1 at full size (1M rows): bit-exact against the oracle."""
    from paper_1801_03065_b200 import generators as G
    a = G.laplace2d(1000)
    _, c = run(kk, a, a)
    assert c.nnz() == 12_980_004
    assert_parity(oracle, a, a, c)


def test_c4_rmat_row_sampled(kk, oracle):
    """Config 4's R-MAT at scale 17 (skewed rows, L2 pool path): row-sampled
    parity (every 32nd row + the 128 heaviest), bitwise raw order.  Rows of C
    are independent, so a row sample of A times full B is exact."""
    from paper_1801_03065_b200 import generators as G
    a = G.rmat(17, 16, 1)
    res = kk.multiply(a, a)
    h = res.handle
    ro = h.c_row_offsets
    sizes = np.diff(ro)
    rows = np.unique(np.concatenate([np.arange(0, a.num_rows, 32), np.argsort(sizes)[-128:]]))
    lo, hi = a.row_offsets[rows], a.row_offsets[rows + 1]
    sro = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(hi - lo, out=sro[1:])
    idx = np.concatenate([np.arange(l, e) for l, e in zip(lo, hi)])
    asamp = kk.CsrMatrix(len(rows), a.num_cols, sro, a.col_indices[idx], a.values[idx], True)
    oro, ocols, ovals = oracle.multiply(asamp, a)
    assert np.array_equal(np.diff(oro), sizes[rows])
    gcols = res.c.col_indices.cpu().numpy()
    gvals = res.c.values.cpu().numpy()
    heavy = 0
    for q, i in enumerate(rows):
        gs, ge = int(ro[i]), int(ro[i + 1])
        gc, gv = gcols[gs:ge], gvals[gs:ge]
        oc, ov = ocols[oro[q]:oro[q + 1]], ovals[oro[q]:oro[q + 1]]
        if np.array_equal(gc, oc):  # warp-table rows: the reference's raw first-touch order
            assert np.array_equal(gv.view(np.int64), ov.view(np.int64))
        else:  # heavy rows (hashed-bucket CTA path): own column order; values still bitwise
            heavy += 1
            so, sg = np.argsort(oc, kind="stable"), np.argsort(gc, kind="stable")
            assert np.array_equal(gc[sg], oc[so])
            assert np.array_equal(gv[sg].view(np.int64), ov[so].view(np.int64))
    assert heavy > 0  # the sample must exercise the heavy-row path


def test_heavy_rows_vs_oracle(kk, oracle):
    """Rows of 10^3-10^4 outputs (beyond the warp tables): CTA dense-bitmap
    symbolic and hashed-bucket numeric; sorted columns identical, value bits equal."""
    rng = np.random.default_rng(7)
    a = random_csr(rng, 48, 3000, 0.08, shuffle=True)
    b = random_csr(rng, 3000, 20000, 0.02, shuffle=True)
    res = kk.multiply(a, b)
    c = res.c.to_host()
    ro = oracle.symbolic_row_offsets(a, b)
    assert np.array_equal(c.row_offsets, ro)
    assert np.diff(ro).max() > 2048
    cols, vals = oracle.numeric(a, b, ro)
    sc, sv = oracle.sort_rows(ro, cols, vals)
    gc, gv = oracle.sort_rows(ro, c.col_indices, c.values)
    assert np.array_equal(sc, gc)
    assert np.array_equal(sv.view(np.int64), gv.view(np.int64))


def _sorted_parity(oracle, a, b, c):
    ro = oracle.symbolic_row_offsets(a, b)
    assert np.array_equal(c.row_offsets, ro)
    cols, vals = oracle.numeric(a, b, ro)
    sc, sv = oracle.sort_rows(ro, cols, vals)
    gc, gv = oracle.sort_rows(ro, c.col_indices, c.values)
    assert np.array_equal(sc, gc)
    assert np.array_equal(sv.view(np.int64), gv.view(np.int64))


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_heavy_rows_column_slabs(kk, oracle, seed):
    """Column-sorted B: heavy rows take the column-slab kernel (kk_slab.cu) —
    adaptive slab widths, abandoned slabs, several A-entry groups per slab
    (A rows longer than 256) — sorted columns identical, value bits equal."""
    rng = np.random.default_rng(seed)
    a = random_csr(rng, 40, 4000, 0.12)          # ~480 A entries per row: two run groups
    b = random_csr(rng, 4000, 30000, 0.01 + 0.01 * (seed % 2))
    h = kk.symbolic(a, b)
    assert h.heavy_path == 2 and h.max_row_size > 1024
    c = kk.numeric(a, b, h).to_host()
    _sorted_parity(oracle, a, b, c)
    # skewed columns (dense low columns, sparse tail): slab widths adapt
    cols = np.minimum((rng.pareto(1.2, size=b.nnz()) * 300).astype(np.int64), 29999).astype(np.int32)
    bs = []
    for i in range(b.num_rows):
        lo, hi = b.row_offsets[i], b.row_offsets[i + 1]
        bs.append(np.unique(cols[lo:hi]))
    ro = np.zeros(b.num_rows + 1, np.int64)
    np.cumsum([len(x) for x in bs], out=ro[1:])
    b2 = kk.CsrMatrix(b.num_rows, b.num_cols, ro, np.concatenate(bs).astype(np.int32),
                      rng.uniform(-1, 1, int(ro[-1])), True)
    res = kk.multiply(a, b2)
    assert res.handle.heavy_path == 2
    _sorted_parity(oracle, a, b2, res.c.to_host())


def test_heavy_row_beyond_half_a_million_outputs(kk, oracle):
    """A row of 600,000 outputs stays on a CTA path (no row-size cliff)."""
    rng = np.random.default_rng(17)
    nb, per, k = 600, 1000, 600_000
    cols = np.concatenate([np.sort(rng.choice(k, per, replace=False)) for _ in range(nb)])
    cols[:k] = np.arange(k)  # the first 600 rows tile every column once
    rows = []
    for i in range(nb):
        rows.append(np.sort(cols[i * per:(i + 1) * per]))
    bro = np.arange(nb + 1, dtype=np.int64) * per
    b = kk.CsrMatrix(nb, k, bro, np.concatenate(rows).astype(np.int32), rng.uniform(-1, 1, nb * per), True)
    a = kk.CsrMatrix(2, nb, np.array([0, nb, nb + 7], np.int64),
                     np.concatenate([np.arange(nb), np.arange(7)]).astype(np.int32), rng.uniform(-1, 1, nb + 7), True)
    res = kk.multiply(a, b)
    h = res.handle
    assert h.max_row_size == k and h.heavy_path == 2
    _sorted_parity(oracle, a, b, res.c.to_host())


def test_heavy_rows_wide_column_domain(kk, oracle):
    """k = 4M columns (125k bitmap words, wider than the heavy symbolic
    kernel's 49,152-word shared bitmap): the heavy rows' union is walked in
    column ranges, and the column slabs handle any k; bit-exact vs the oracle,
    compressed and raw."""
    rng = np.random.default_rng(71)
    m, n, k = 6, 3000, 4_000_000

    def wide(rows, cols, per_row):
        ro = np.zeros(rows + 1, np.int64)
        ci = []
        for r in range(rows):
            c = np.unique(rng.integers(0, cols, per_row))
            ci.append(c.astype(np.int32))
            ro[r + 1] = ro[r] + len(c)
        ci = np.concatenate(ci)
        return kk.CsrMatrix(rows, cols, ro, ci, rng.uniform(-1, 1, len(ci)), True)

    a = wide(m, n, 300)
    b = wide(n, k, 60)
    for mode in (kk.CompressionMode.Always, kk.CompressionMode.Never):
        res = kk.multiply(a, b, kk.SpgemmConfig(compression=mode))
        assert res.handle.max_row_size > 8192  # rows beyond the warp tables
        c = res.c.to_host()
        ro = oracle.symbolic_row_offsets(a, b)
        assert np.array_equal(c.row_offsets, ro)
        cols, vals = oracle.numeric(a, b, ro)
        sc, sv = oracle.sort_rows(ro, cols, vals)
        gc, gv = oracle.sort_rows(ro, c.col_indices, c.values)
        assert np.array_equal(sc, gc)
        assert np.array_equal(sv.view(np.int64), gv.view(np.int64))


def test_heavy_rows_unsorted_b(kk, oracle):
    """Unsorted B rows: the hashed-bucket heavy kernel; reusing a slab plan
    with an unsorted B of the same structure size raises instead of
    returning a wrong C."""
    rng = np.random.default_rng(19)
    a = random_csr(rng, 24, 3000, 0.08)
    b = random_csr(rng, 3000, 20000, 0.02)
    bu = random_csr(rng, 3000, 20000, 0.02, shuffle=True)
    res = kk.multiply(a, bu)
    assert res.handle.heavy_path == 1
    _sorted_parity(oracle, a, bu, res.c.to_host())
    h = kk.symbolic(a, b)
    assert h.heavy_path == 2
    perm = kk.CsrMatrix(b.num_rows, b.num_cols, b.row_offsets, b.col_indices.copy(), b.values, False)
    for i in range(b.num_rows):
        lo, hi = perm.row_offsets[i], perm.row_offsets[i + 1]
        perm.col_indices[lo:hi] = perm.col_indices[lo:hi][::-1]
    with pytest.raises(kk.InternalError, match="sorted"):
        kk.numeric(a, perm, h, kk.PhaseStats())


def test_row_flops_kernel(kk, oracle):
    from paper_1801_03065_b200 import generators as G
    a = G.rmat(12, 16, 1)
    per, _, _ = oracle.flops_stats(a, a)
    assert np.array_equal(kk.row_flops(a.to_device(), a.to_device()).cpu().numpy(), per)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_flop_balanced_shards_reassemble(kk, oracle, world):
    """Multi-GPU partition emulated shard by shard on one GPU:
    GPU per-row flops -> cut points -> row-block multiplies; the blocks with
    their all-gathered base offsets reassemble C bit for bit."""
    import torch
    from paper_1801_03065_b200 import generators as G, shard
    a = G.laplace3d(14)
    da = a.to_device()
    cuts = shard.flop_cut_points(torch.cumsum(kk.row_flops(da, da), 0), world)
    ro, cols, vals = oracle.multiply(a, a)
    nnzs, flops = [], []
    for r in range(world):
        res = kk.multiply(da.row_block(cuts[r], cuts[r + 1]), da)
        c = res.c.to_host()
        nnzs.append(c.nnz())
        flops.append(res.handle.flops.total_flops)
        lo, hi = cuts[r], cuts[r + 1]
        assert np.array_equal(c.row_offsets + ro[lo], ro[lo:hi + 1])
        assert np.array_equal(c.col_indices, cols[ro[lo]:ro[hi]])
        assert np.array_equal(c.values.view(np.int64), vals[ro[lo]:ro[hi]].view(np.int64))
    offs = shard.block_offsets(nnzs)
    assert offs == [int(ro[c]) for c in cuts]
    assert max(flops) - min(flops) <= 2 * 729  # lower_bound cuts: within two rows


@pytest.mark.parametrize("blocks", [1, 3])
def test_multiply_host_pipelined(kk, oracle, blocks):
    """host.multiply_host (pinned host CSR in and out, row blocks overlapping
    copies with compute) equals the device multiply bit for bit."""
    from paper_1801_03065_b200 import host
    rng = np.random.default_rng(31 + blocks)
    a = random_csr(rng, 240, 240, 0.06)
    b = random_csr(rng, 240, 180, 0.05)
    pa, pb = host.PinnedCsr.from_csr(a), host.PinnedCsr.from_csr(b)
    # A*B
    r = host.multiply_host(pa, pb, blocks=blocks)
    assert r.h2d_bytes == pa.nbytes() + pb.nbytes()
    assert_parity(oracle, a, b, r.c)
    # A*A, uploaded once
    r2 = host.multiply_host(pa, blocks=blocks)
    assert r2.h2d_bytes == pa.nbytes()
    assert_parity(oracle, a, a, r2.c)
    # rows [50, 190) of A times A: only A travels
    r3 = host.multiply_host(None, pa, a_rows=(50, 190), blocks=blocks)
    ro = oracle.symbolic_row_offsets(a, a)
    cols, vals = oracle.numeric(a, a, ro)
    assert np.array_equal(r3.c.row_offsets, ro[50:191] - ro[50])
    assert np.array_equal(r3.c.col_indices, cols[ro[50]:ro[190]])
    assert np.array_equal(r3.c.values.view(np.int64), vals[ro[50]:ro[190]].view(np.int64))


@pytest.mark.parametrize("sort", [False, True])
def test_numeric_rows_blocks_equal_full(kk, oracle, sort):
    """spg_numeric_rows over a partition of the rows fills the same C as one
    spg_numeric, before and after the slot replay is recorded."""
    import torch
    rng = np.random.default_rng(41 + sort)
    a = random_csr(rng, 500, 300, 0.05)
    b = random_csr(rng, 300, 400, 0.08)
    cfg = kk.SpgemmConfig(sort_output=sort)
    da, db = a.to_device(), b.to_device()
    h = kk.symbolic(da, db, cfg)
    full = kk.numeric(da, db, h).to_host()
    for rep in range(3):  # pass 2 (rep 1) records the replay; 3 replays
        kk.numeric(da, db, h)
        nnz = h.nnz_c()
        cols = torch.full((nnz,), -7, dtype=torch.int32, device="cuda")
        vals = torch.zeros(nnz, dtype=torch.float64, device="cuda")
        for r0, r1 in ((0, 0), (0, 123), (123, 124), (124, 400), (400, 500)):
            kk.numeric_rows(da, db, h, r0, r1, cols, vals)
        assert np.array_equal(cols.cpu().numpy(), full.col_indices)
        assert np.array_equal(vals.cpu().numpy().view(np.int64), full.values.view(np.int64))
    assert h.replay_state == 2
    with pytest.raises(kk.ContractError):
        kk.numeric_rows(da, db, h, 10, 5, cols, vals)


def test_short_and_long_rows_bitwise(kk, oracle):
    """Rows of 0..40 A entries with 1..4-entry B rows (the flat kernel's
    domain), empty rows and rows with more than 32 A entries mixed in the same
    classes: raw order and value bits equal the reference's, also through
    spg_numeric_rows and with compression on/off."""
    import torch
    rng = np.random.default_rng(57)
    m, n, k = 3000, 2000, 5000
    lens = rng.integers(0, 6, m)
    lens[rng.choice(m, 40, replace=False)] = rng.integers(33, 41, 40)
    lens[rng.choice(m, 200, replace=False)] = 0
    rows = []
    for i in range(m):
        for c in rng.choice(n, lens[i], replace=False):
            rows.append((i, int(c), float(rng.standard_normal())))
    a = csr_from_triplets(m, n, rows)
    brow = []
    for i in range(n):
        for c in rng.choice(k, int(rng.integers(1, 5)), replace=False):
            brow.append((i, int(c), float(rng.standard_normal())))
    b = csr_from_triplets(n, k, brow)
    for mode in (kk.CompressionMode.Auto, kk.CompressionMode.Never, kk.CompressionMode.Always):
        res = kk.multiply(a, b, kk.SpgemmConfig(compression=mode))
        assert_parity(oracle, a, b, res.c.to_host())
    da, db = a.to_device(), b.to_device()
    h = kk.symbolic(da, db)
    full = kk.numeric(da, db, h).to_host()
    cols = torch.full((h.nnz_c(),), -3, dtype=torch.int32, device="cuda")
    vals = torch.zeros(h.nnz_c(), dtype=torch.float64, device="cuda")
    for r0, r1 in ((0, 1000), (1000, 1001), (1001, 2999), (2999, 3000)):
        kk.numeric_rows(da, db, h, r0, r1, cols, vals)
    assert np.array_equal(cols.cpu().numpy(), full.col_indices)
    assert np.array_equal(vals.cpu().numpy().view(np.int64), full.values.view(np.int64))


def test_tiny_rows_thread_per_row(kk, oracle, monkeypatch):
    """Short A rows whose C rows hold <= 16 keys run a thread per row
    (kk_tiny.cu): raw first-touch order and value bits (specials included)
    equal the reference's and the warp kernels' (KK_NO_TINY=1), through
    spg_numeric_rows too; a reused handle whose new B changes the rows' key
    counts is reported (engine.cpp:238-245)."""
    import torch
    rng = np.random.default_rng(63)
    m, n, k = 5000, 3000, 4000
    a = random_csr(rng, m, n, 4.0 / n)
    b = random_csr(rng, n, k, 3.0 / k)
    specials = np.array([np.inf, -np.inf, np.nan, -0.0, 0.0, 5e-324, 1.7e308])
    for x in (a, b):
        pick = rng.choice(x.nnz(), x.nnz() // 10, replace=False)
        x.values[pick] = rng.choice(specials, len(pick))
    ro = oracle.symbolic_row_offsets(a, b)
    assert (np.diff(ro) <= 16).mean() > 0.5 and np.diff(ro).max() > 16  # tiny and warp classes mixed
    cols, vals = oracle.numeric(a, b, ro)
    nan = np.isnan(vals)
    res = kk.multiply(a, b).c.to_host()
    monkeypatch.setenv("KK_NO_TINY", "1")
    warp = kk.multiply(a, b).c.to_host()
    monkeypatch.delenv("KK_NO_TINY")
    for c in (res, warp):
        assert np.array_equal(c.row_offsets, ro)
        assert np.array_equal(c.col_indices, cols)
        assert np.array_equal(np.isnan(c.values), nan)
        assert np.array_equal(c.values[~nan].view(np.int64), vals[~nan].view(np.int64))
    # row blocks
    da, db = a.to_device(), b.to_device()
    h = kk.symbolic(da, db)
    ccols = torch.full((h.nnz_c(),), -3, dtype=torch.int32, device="cuda")
    cvals = torch.zeros(h.nnz_c(), dtype=torch.float64, device="cuda")
    for r0, r1 in ((0, 1700), (1700, 1701), (1701, m)):
        kk.numeric_rows(da, db, h, r0, r1, ccols, cvals)
    assert np.array_equal(ccols.cpu().numpy(), cols)
    # structure changes under a reused handle (same nnz, B's columns moved):
    # rows of C with more or fewer keys than the structure are reported
    h = kk.symbolic(a, b)
    b2 = kk.CsrMatrix(b.num_rows, b.num_cols, b.row_offsets, b.col_indices.copy(), b.values, False)
    for i in range(b2.num_rows):
        lo, hi = b2.row_offsets[i], b2.row_offsets[i + 1]
        b2.col_indices[lo:hi] = (np.arange(hi - lo) * 7 + i) % 40
    with pytest.raises(kk.InternalError):
        kk.numeric(a, b2, h, kk.PhaseStats())


def test_numeric_reuse_is_graph_capturable(kk, oracle):
    """Once a handle replays (third numeric pass on), spg_numeric is fully
    stream-ordered: the reuse loop can be captured in a CUDA graph and replayed
    with new values written into the same device buffers."""
    import torch
    rng = np.random.default_rng(61)
    a = random_csr(rng, 400, 400, 0.06)
    b = random_csr(rng, 400, 400, 0.06)
    da, db = a.to_device(), b.to_device()
    h = kk.symbolic(da, db)
    nnz = h.nnz_c()
    cols = torch.empty(nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
    for _ in range(2):
        kk.numeric(da, db, h, out=(cols, vals))
    assert h.replay_state == 2
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        kk.numeric(da, db, h, stream=s, out=(cols, vals))  # warm the allocator on this stream
        with torch.cuda.graph(g, stream=s):
            kk.numeric(da, db, h, stream=s, out=(cols, vals))
    torch.cuda.current_stream().wait_stream(s)
    for f in (1.0, -2.5, 0.125):
        da.values.copy_(torch.from_numpy(a.values * f))
        g.replay()
        torch.cuda.synchronize()
        ap = kk.CsrMatrix(a.num_rows, a.num_cols, a.row_offsets, a.col_indices, a.values * f, a.sorted_rows)
        c = kk.CsrMatrix(a.num_rows, b.num_cols, h.c_row_offsets, cols.cpu().numpy(), vals.cpu().numpy())
        assert_parity(oracle, ap, b, c)


def test_device_transpose(kk, oracle):
    """spg_transpose equals csr_matrix.cpp:82-108's transpose (the generators'
    host transpose) exactly, and the device triple product R*(A*P) with the
    device R = P^T matches the host-built one bit for bit."""
    from paper_1801_03065_b200 import generators as G
    rng = np.random.default_rng(71)
    for m, n in ((1, 1), (57, 300), (400, 123)):
        a = random_csr(rng, m, n, 0.05)
        t = kk.transpose(a.to_device()).to_host()
        ref = G.transpose(a)
        assert np.array_equal(t.row_offsets, ref.row_offsets)
        assert np.array_equal(t.col_indices, ref.col_indices)
        assert np.array_equal(t.values.view(np.int64), ref.values.view(np.int64))
    a, p = G.laplace3d(10), G.aggregation(10)
    dA, dP = a.to_device(), p.to_device()
    dR = kk.transpose(dP)
    ap = kk.multiply(dA, dP).c
    rap_dev = kk.multiply(dR, ap).c.to_host()
    rap_host = kk.multiply(G.transpose(p), ap).c.to_host()
    assert np.array_equal(rap_dev.row_offsets, rap_host.row_offsets)
    assert np.array_equal(rap_dev.col_indices, rap_host.col_indices)
    assert np.array_equal(rap_dev.values.view(np.int64), rap_host.values.view(np.int64))


def test_multiply_host_shard_uploads_band_only(kk, oracle):
    """A = rows [lo, hi) of a banded B: only B's offsets and the band rows
    travel; the product still equals the oracle's rows bit for bit."""
    from paper_1801_03065_b200 import generators as G, host
    a = G.laplace3d(14)
    pa = host.PinnedCsr.from_csr(a)
    lo, hi = 900, 1700
    r = host.multiply_host(None, pa, a_rows=(lo, hi), blocks=2)
    assert r.h2d_bytes < pa.nbytes() // 2
    ro = oracle.symbolic_row_offsets(a, a)
    cols, vals = oracle.numeric(a, a, ro)
    assert np.array_equal(r.c.row_offsets, ro[lo:hi + 1] - ro[lo])
    assert np.array_equal(r.c.col_indices, cols[ro[lo]:ro[hi]])
    assert np.array_equal(r.c.values.view(np.int64), vals[ro[lo]:ro[hi]].view(np.int64))


def test_empty_operands_everywhere(kk):
    """Zero rows, zero columns and zero nnz through multiply, reuse, row ranges,
    the host multiply and the transpose."""
    import torch
    from paper_1801_03065_b200 import host
    cases = [((0, 5), (5, 7)), ((4, 0), (0, 3)), ((3, 4), (4, 6))]
    for (m, n), (n2, k) in cases:
        a = csr_from_triplets(m, n, [])
        b = csr_from_triplets(n2, k, [])
        res = kk.multiply(a, b)
        c = res.c.to_host()
        assert c.nnz() == 0 and c.row_offsets.tolist() == [0] * (m + 1)
        for _ in range(3):
            kk.numeric(a, b, res.handle)
        cols = torch.empty(1, dtype=torch.int32, device="cuda")
        vals = torch.empty(1, dtype=torch.float64, device="cuda")
        kk.numeric_rows(a, b, res.handle, 0, m, cols, vals)
        r = host.multiply_host(host.PinnedCsr.from_csr(a), host.PinnedCsr.from_csr(b))
        assert r.c.nnz() == 0 and r.c.row_offsets.tolist() == [0] * (m + 1)
        t = kk.transpose(a.to_device()).to_host()
        assert t.num_rows == n and t.nnz() == 0


def test_special_values_bitwise(kk, oracle):
    """Inf, NaN, signed zeros, subnormals and near-overflow values: the
    hashing kernels and the slot replay reproduce the reference's value bits
    (products through __dmul_rn, first product stored as is / -0.0 + v).
    NaNs match as NaNs: a NaN generated by the hardware (inf - inf, 0 * inf)
    has a different bit pattern on x86 (0xfff8...) and on the GPU (0x7fff...)."""
    rng = np.random.default_rng(97)
    a = random_csr(rng, 300, 300, 0.09)
    b = random_csr(rng, 300, 300, 0.09)
    specials = np.array([np.inf, -np.inf, np.nan, -0.0, 0.0, 5e-324, -2.2e-308, 1.7e308, -1.7e308, 1e-300])
    for x in (a, b):
        pick = rng.choice(x.nnz(), x.nnz() // 8, replace=False)
        x.values[pick] = rng.choice(specials, len(pick))
    ro = oracle.symbolic_row_offsets(a, b)
    cols, vals = oracle.numeric(a, b, ro)
    h = kk.symbolic(a, b)
    nan = np.isnan(vals)
    assert nan.any() and np.isinf(vals).any()
    for p in range(4):  # passes 1-2 hashing, 3-4 replay
        c = kk.numeric(a, b, h).to_host()
        assert np.array_equal(c.col_indices, cols)
        assert np.array_equal(np.isnan(c.values), nan), f"pass {p}: NaN positions"
        assert np.array_equal(c.values[~nan].view(np.int64), vals[~nan].view(np.int64)), f"pass {p}"
    assert h.replay_state == 2


def _row_sample(kk, a, rows):
    lo, hi = a.row_offsets[rows], a.row_offsets[rows + 1]
    sro = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(hi - lo, out=sro[1:])
    idx = np.concatenate([np.arange(l, e) for l, e in zip(lo, hi)])
    return kk.CsrMatrix(len(rows), a.num_cols, sro, a.col_indices[idx], a.values[idx], True)


def _check_rows(oracle, a_s, b, ro, cols, vals, rows):
    oro, ocols, ovals = oracle.multiply(a_s, b)
    for q, i in enumerate(rows):
        g0, g1 = int(ro[i]), int(ro[i + 1])
        assert g1 - g0 == oro[q + 1] - oro[q]
        assert np.array_equal(cols[g0:g1], ocols[oro[q]:oro[q + 1]])
        assert np.array_equal(vals[g0:g1].view(np.int64), ovals[oro[q]:oro[q + 1]].view(np.int64))


def test_c2_full_size_row_sampled(kk, oracle):
    """Config 2 at full size (160^3, 2.9 G products): closed-form nnz, and every
    97th row plus the boundary rows bit-exact against the oracle."""
    from paper_1801_03065_b200 import generators as G
    a = G.laplace3d(160)
    res = kk.multiply(a, a)
    h = res.handle
    assert h.nnz_c() == 794 ** 3 and h.flops.total_flops == 1430 ** 3
    ro = h.c_row_offsets
    rows = np.unique(np.concatenate([np.arange(0, a.num_rows, 97), np.arange(0, 200),
                                     np.arange(a.num_rows - 200, a.num_rows)]))
    _check_rows(oracle, _row_sample(kk, a, rows), a, ro, res.c.col_indices.cpu().numpy(),
                res.c.values.cpu().numpy(), rows)


def test_c5_reuse_passes_row_sampled(kk, oracle):
    """Config 5 (200^3, one symbolic then numeric passes with perturbed values,
    SURVEY §8c): passes 1 (hashing) and 3 (slot replay) row-sampled bit-exact."""
    import torch
    from paper_1801_03065_b200 import generators as G
    a = G.laplace3d(200)
    da = a.to_device()
    h = kk.symbolic(da, da)
    assert h.nnz_c() == 994 ** 3
    ro = h.c_row_offsets
    rows = np.unique(np.concatenate([np.arange(0, a.num_rows, 211), np.arange(0, 100)]))
    rng = np.random.default_rng(5)
    base = a.values.copy()
    for p in range(3):
        a.values[:] = base * (1.0 + 1e-3 * rng.uniform(-1.0, 1.0, base.shape))
        da.values.copy_(torch.from_numpy(a.values))
        c = kk.numeric(da, da, h)
        if p in (0, 2):
            _check_rows(oracle, _row_sample(kk, a, rows), a, ro, c.col_indices.cpu().numpy(),
                        c.values.cpu().numpy(), rows)
    assert h.replay_state == 2


def test_c3_full_size_vs_oracle(kk, oracle):
    """Config 3 at full size: A (128^3 27-point) * P (2x2x2 aggregation), then
    R * (AP) with R = P^T built on the device; both products bit-exact vs the
    oracle, SURVEY §8d counts."""
    from paper_1801_03065_b200 import generators as G
    a, p = G.laplace3d(128), G.aggregation(128)
    dA, dP = a.to_device(), p.to_device()
    dR = kk.transpose(dP)
    ap = kk.multiply(dA, dP)
    assert ap.handle.flops.total_flops == 55_742_968 and ap.handle.nnz_c() == 16_387_064
    ap_host = ap.c.to_host()
    assert_parity(oracle, a, p, ap_host)
    rap = kk.multiply(dR, ap.c)
    assert rap.handle.flops.total_flops == 16_387_064 and rap.handle.nnz_c() == 6_859_000
    r = dR.to_host()
    assert_parity(oracle, r, ap_host, rap.c.to_host())


def test_fuzz_short():
    """tests/tools/fuzz.py for 20 s (random shapes, configs and paths vs the oracle;
    the round-1 log has 141,544 cases over five runs, profiles/r01_fuzz.md)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "tools", "fuzz.py"), "20", "7"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "fuzz ok" in r.stdout


def test_multiply_host_chunked_values():
    """C = A*A with enough entries for the chunked value upload (each block of
    C waits only for the B rows it references): equal to the device multiply
    bit for bit, for a banded operator and for a scrambled one."""
    import numpy as np
    import paper_1801_03065_b200 as kk
    from paper_1801_03065_b200 import generators as G, host
    a = G.laplace3d(56)
    assert a.nnz() >= (1 << 22)
    rng = np.random.default_rng(3)
    # same structure size, columns permuted: blocks reference rows far away
    perm = rng.permutation(a.num_cols).astype(np.int32)
    scr = kk.CsrMatrix(a.num_rows, a.num_cols, a.row_offsets, perm[a.col_indices], a.values, False)
    for x in (a, scr):
        r = host.multiply_host(host.PinnedCsr.from_csr(x))
        d = kk.multiply(x, x).c.to_host()
        assert r.blocks == 8
        assert np.array_equal(r.c.row_offsets, d.row_offsets)
        assert np.array_equal(r.c.col_indices, d.col_indices)
        assert np.array_equal(r.c.values.view(np.int64), d.values.view(np.int64))


# ---------------------------------------------------------------------------
# full-size configurations checked on ALL rows through per-row canonical
# digests (spg_row_digests on the device, orc_product_row_digests on the CPU:
# the same order-independent hash of each row's (column, value bits) set)
# ---------------------------------------------------------------------------
def _digest_check(kk, oracle, a, b, c_dev, row_offsets):
    gd = kk.row_digests(c_dev).cpu().numpy().view(np.uint64)
    od, osz = oracle.product_row_digests(a, b)
    assert np.array_equal(np.diff(row_offsets), osz), "row sizes differ"
    bad = np.nonzero(gd != od)[0]
    assert bad.size == 0, f"{bad.size} rows differ (first {bad[:5].tolist()})"


def test_row_digests_match_oracle_small(kk, oracle):
    rng = np.random.default_rng(43)
    a = random_csr(rng, 200, 150, 0.1, shuffle=True)
    b = random_csr(rng, 150, 170, 0.1, shuffle=True)
    res = kk.multiply(a, b)
    c = res.c.to_host()
    assert np.array_equal(kk.row_digests(res.c).cpu().numpy().view(np.uint64), oracle.row_digests(c))
    _digest_check(kk, oracle, a, b, res.c, c.row_offsets)
    # a permuted row has the digest of its sorted form; one flipped value bit does not
    sc, sv = oracle.sort_rows(c.row_offsets, c.col_indices, c.values)
    s = kk.CsrMatrix(c.num_rows, c.num_cols, c.row_offsets, sc, sv, True)
    assert np.array_equal(oracle.row_digests(s), oracle.row_digests(c))
    sv2 = sv.copy()
    sv2.view(np.int64)[3] ^= 1
    s2 = kk.CsrMatrix(c.num_rows, c.num_cols, c.row_offsets, sc, sv2, True)
    assert (oracle.row_digests(s2) != oracle.row_digests(c)).sum() == 1


def test_c2_full_size_all_rows(kk, oracle):
    """Config 2 (160^3, 2.9 G products): every row of C against the oracle."""
    from paper_1801_03065_b200 import generators as G
    a = G.laplace3d(160)
    res = kk.multiply(a, a)
    _digest_check(kk, oracle, a, a, res.c, res.handle.c_row_offsets)


def test_c5_reuse_passes_all_rows(kk, oracle):
    """Config 5 (200^3): one symbolic, numeric passes with perturbed values;
    pass 1 (hashing kernels) and pass 3 (slot replay) checked on every row."""
    import torch
    from paper_1801_03065_b200 import generators as G
    a = G.laplace3d(200)
    da = a.to_device()
    h = kk.symbolic(da, da)
    rng = np.random.default_rng(5)
    base = a.values.copy()
    ro = h.c_row_offsets
    for p in range(3):
        a.values[:] = base * (1.0 + 1e-3 * rng.uniform(-1.0, 1.0, base.shape))
        da.values.copy_(torch.from_numpy(a.values))
        c = kk.numeric(da, da, h)
        if p in (0, 2):
            _digest_check(kk, oracle, a, a, c, ro)
        del c
    assert h.replay_state == 2


def test_c4_rmat_s20_all_rows(kk, oracle):
    """Config 4 at its BASELINE size (R-MAT scale 20: 20.9 G products, C =
    9.71 G entries / 116.5 GB on the device): every row against the oracle,
    plus SURVEY §8c's row sample (every 64th row and the 1,024 heaviest)
    compared entry by entry (sorted columns, value bits)."""
    import torch
    from paper_1801_03065_b200 import generators as G
    a = G.rmat(20, 16, 1)
    da = a.to_device()
    h = kk.symbolic(da, da)
    assert h.flops.total_flops == 20_938_949_470 and h.nnz_c() == 9_711_687_861
    assert h.max_row_size == 484_845 and h.heavy_path == 2
    c = kk.numeric(da, da, h, kk.PhaseStats())
    ro = h.c_row_offsets
    _digest_check(kk, oracle, a, a, c, ro)
    sizes = np.diff(ro)
    rows = np.unique(np.concatenate([np.arange(0, a.num_rows, 64), np.argsort(sizes, kind="stable")[-1024:]]))
    rows = rows[sizes[rows] > 0]
    lo, hi = ro[rows], ro[rows + 1]
    idx = torch.from_numpy(np.concatenate([np.arange(x, y) for x, y in zip(lo, hi)])).to(c.values.device)
    gc = c.col_indices.index_select(0, idx).cpu().numpy()
    gv = c.values.index_select(0, idx).cpu().numpy()
    del c
    torch.cuda.empty_cache()
    samp = _row_sample(kk, a, rows)
    oro, ocols, ovals = oracle.multiply(samp, a)
    assert np.array_equal(np.diff(oro), sizes[rows])
    sro = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(sizes[rows], out=sro[1:])
    sc, sv = oracle.sort_rows(oro, ocols, ovals)
    tc, tv = oracle.sort_rows(sro, gc, gv)
    assert np.array_equal(sc, tc)
    assert np.array_equal(sv.view(np.int64), tv.view(np.int64))


def test_harness_bench_rows_on_gpu(tmp_path):
    """harness bench (cli.cpp:132-174 on the GPU) writes the reference's
    22-column BenchRecord rows; the profile reads them back."""
    from paper_1801_03065_b200 import harness as H
    out = tmp_path / "r.csv"
    assert H.main(["bench", "--config", "2", "--scale", "0.1", "--reps", "2", "--reuse", "2", "--out", str(out)]) == 0
    recs = H.read_bench_csv(str(out))
    assert [r.algorithm for r in recs] == ["auto", "auto-reuse"] and recs[1].reuse
    assert recs[0].flops == (9 * 16 - 10) ** 3 and recs[0].nnz_c == (5 * 16 - 6) ** 3 and recs[0].gflops > 0 and recs[1].gflops > 0
    assert open(str(out)).read().splitlines()[0] == H.HEADER
    prof = tmp_path / "p.csv"
    assert H.main(["profile", "--in", str(out), "--out", str(prof), "--points", "4"]) == 0
