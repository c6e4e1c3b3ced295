"""GPU checks of the C-ABI boundary contract (include/swsearch.h):

* device memory comes from the caller's allocator hooks (torch's caching
  allocator here), and no search allocates after sw_db_create -- the paper
  pre-allocates its buffers and reuses them for the whole search;
* sw_search_async refuses queries beyond the reserved capacity instead of
  allocating, and sw_db_reserve grows it;
* one handle orders its searches whatever streams they are enqueued on
  (async on a torch stream followed by a blocking search, no host sync);
* handles used from several threads with different query lengths stay exact
  (the dynamic-shared-memory attribute is only ever raised).
Every score is compared with the oracle.
"""
import threading

import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum62, matrix32, random_db, stream_key
from swdata.synth import gen_residues

pytestmark = pytest.mark.gpu
B62 = matrix32(blosum62())


def _query(m, seed=0):
    return gen_residues(stream_key(seed, "boundary-query", m), 0, m)


def _db(seed=3, n=3000):
    rng = np.random.default_rng(seed)
    return random_db(seed, np.concatenate([rng.integers(0, 800, n), [4000, 5200, 0, 1]]))


def test_torch_allocator_backs_every_buffer_and_searches_allocate_nothing():
    import torch
    db = _db()
    qs = [_query(m, m) for m in (1, 37, 464, 1000, 2100)]
    g = sw.Database.from_synth(db, device=0, allocator="torch", max_qlen=2500, max_k=64)
    a = g.allocator
    info0 = g.info()
    assert a.n_alloc > 0 and info0["n_device_allocs"] == a.n_alloc and a.n_free == 0
    assert info0["device_bytes"] == sum(a.live.values())
    n0 = a.n_alloc
    stream = torch.cuda.Stream()
    d_sc = torch.empty(db.n_seqs, dtype=torch.int32, device="cuda")
    d_ti = torch.empty(64, dtype=torch.int64, device="cuda")
    d_ts = torch.empty(64, dtype=torch.int32, device="cuda")
    for q in qs:
        for k in (1, 10, 64):
            g.search_async(q, B62, 2, 12, k, d_sc, d_ti, d_ts, stream=stream)
            stream.synchronize()
            ref = oracle.db_scores(q, db, B62, 2, 12)
            assert np.array_equal(d_sc.cpu().numpy(), ref)
            ti, ts = oracle.topk(ref, k)
            assert np.array_equal(d_ti[:k].cpu().numpy(), ti) and np.array_equal(d_ts[:k].cpu().numpy(), ts)
        r = g.search(q, B62, 2, 12, k=7)                    # blocking path, within capacity
        assert np.array_equal(r.scores, oracle.db_scores(q, db, B62, 2, 12))
    assert a.n_alloc == n0 and g.info()["n_device_allocs"] == n0, "a search allocated device memory"
    g.close()
    assert a.n_free == a.n_alloc and not a.live


def test_async_beyond_capacity_is_refused_then_reserved():
    import torch
    db = _db(5, 500)
    g = sw.Database.from_synth(db, device=0, max_qlen=100, max_k=8)
    d_sc = torch.empty(db.n_seqs, dtype=torch.int32, device="cuda")
    d_ti = torch.empty(16, dtype=torch.int64, device="cuda")
    d_ts = torch.empty(16, dtype=torch.int32, device="cuda")
    q = _query(300, 1)
    with pytest.raises(sw.SwError) as e:
        g.search_async(q, B62, 2, 12, 8, d_sc, d_ti, d_ts)
    assert e.value.code == sw.SW_EINVAL and "capacity" in str(e.value)
    with pytest.raises(sw.SwError):
        g.search_async(q[:50], B62, 2, 12, 16, d_sc, d_ti, d_ts)
    n0 = g.info()["n_device_allocs"]
    g.reserve(300, 16)
    assert g.info()["max_qlen"] == 300 and g.info()["max_k"] == 16 and g.info()["n_device_allocs"] > n0
    g.search_async(q, B62, 2, 12, 16, d_sc, d_ti, d_ts)
    torch.cuda.synchronize()
    ref = oracle.db_scores(q, db, B62, 2, 12)
    assert np.array_equal(d_sc.cpu().numpy(), ref)
    # the blocking call grows the capacity itself
    r = g.search(_query(700, 2), B62, 2, 12, k=40)
    assert np.array_equal(r.scores, oracle.db_scores(_query(700, 2), db, B62, 2, 12))
    assert g.info()["max_qlen"] == 700 and g.info()["max_k"] == 40
    g.close()


def test_async_on_torch_stream_then_blocking_search_without_host_sync():
    """sw_search used to enqueue on its own stream without waiting for an
    async search still running on another stream (shared per-search buffers)."""
    import torch
    db = _db(8, 20000)
    qa, qb = _query(1500, 11), _query(200, 12)
    stream = torch.cuda.Stream()
    d_sc = torch.empty(db.n_seqs, dtype=torch.int32, device="cuda")
    with sw.Database.from_synth(db, device=0) as g:
        for _ in range(3):
            g.search_async(qa, B62, 2, 12, 5, d_sc, None, None, stream=stream)   # long search in flight
            r = g.search(qb, B62, 2, 12, k=5)                                   # no sync in between
            stream.synchronize()
            assert np.array_equal(r.scores, oracle.db_scores(qb, db, B62, 2, 12))
            assert np.array_equal(d_sc.cpu().numpy(), oracle.db_scores(qa, db, B62, 2, 12))


def test_two_handles_from_two_threads_with_different_query_lengths():
    """the per-kernel max-dynamic-smem attribute is process-wide; it is
    now only raised, so a concurrent launch never sees it lowered."""
    dbs = [_db(21, 1500), _db(22, 1500)]
    qs = [[_query(m, 30 + m) for m in (50, 1900, 300, 1200)], [_query(m, 40 + m) for m in (1700, 80, 900, 20)]]
    refs = [[oracle.db_scores(q, d, B62, 2, 12) for q in ql] for d, ql in zip(dbs, qs)]
    errors = []

    def work(t):
        try:
            with sw.Database.from_synth(dbs[t], device=0) as g:
                for rep in range(3):
                    for q, ref in zip(qs[t], refs[t]):
                        r = g.search(q, B62, 2, 12, k=3)
                        if not np.array_equal(r.scores, ref):
                            errors.append((t, q.size))
        except Exception as e:   # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(t,)) for t in (0, 1)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors


class _FailingAllocator(sw.TorchAllocator):
    """torch-backed hooks that refuse the (fail_at+1)-th allocation (fault injection)."""

    def __init__(self, device, fail_at):
        import torch
        super().__init__(device)
        self.fail_at = fail_at
        inner = self.alloc_fn

        def _alloc(nbytes, ctx):
            if self.n_alloc >= self.fail_at:
                return None
            return inner(nbytes, ctx)

        self.alloc_fn = sw.ALLOC_FN(_alloc)
        self._keep = inner


@pytest.mark.parametrize("residency", [0, 1])
def test_allocation_failure_at_every_step_of_create_is_clean(residency):
    """Every device allocation of sw_db_create / sw_db_reserve in turn refused: SW_ENOMEM, no handle, and
    every buffer that was handed out is given back (no leak); one more allocation and create succeeds."""
    db = _db(31, 300)
    total = None
    ok = sw.TorchAllocator(0)
    with sw.Database.from_synth(db, device=0, allocator=ok, residency=residency) as g:
        total = g.info()["n_device_allocs"]
    assert total and ok.n_free == ok.n_alloc == total
    for fail_at in range(total):
        a = _FailingAllocator(0, fail_at)
        with pytest.raises(sw.SwError) as e:
            sw.Database.from_synth(db, device=0, allocator=a, residency=residency)
        assert e.value.code == sw.SW_ENOMEM, (fail_at, str(e.value))
        assert a.n_alloc == fail_at and a.n_free == a.n_alloc and not a.live, fail_at
    a = _FailingAllocator(0, total)
    with sw.Database.from_synth(db, device=0, allocator=a, residency=residency) as g:
        q = _query(120, 5)
        assert np.array_equal(g.search(q, B62, 2, 12, k=3).scores, oracle.db_scores(q, db, B62, 2, 12))
        with pytest.raises(sw.SwError) as e:            # growing past the hooks' budget fails cleanly too
            g.reserve(20000, 5000)
        assert e.value.code == sw.SW_ENOMEM
        r = g.search(q, B62, 2, 12, k=3)                 # the handle still works within its old capacity
        assert np.array_equal(r.scores, oracle.db_scores(q, db, B62, 2, 12))
    assert a.n_free == a.n_alloc and not a.live
