"""GPU parity of the dense-run join paths (k_dense_flat / k_dense_flat1 and
k_dense_join, csrc/merge_join.cu):
private runs whose keys step by one take it, every other run the merge walk.
Per (private run, public run) pair the record must equal the reference's
interpolation search plus merge_join_run (_kernels.py:287-408) on the same
run -- count, max, checksum, start, probes, end, examined -- and a public run
out of order must raise the pair's order flag.  Run with ``pytest -m gpu``."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1207_0145_b200 import _lib  # noqa: E402
from paper_1207_0145_b200 import device as D  # noqa: E402
from oracle import oracle as orc  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture(autouse=True, params=["streamed", "staged"])
def dense_path(request, monkeypatch):
    """every case through both dense kernels: the streamed k_dense_flat[1]
    (default) and the staged k_dense_join (MPSM_DENSE_FLAT=0)"""
    if request.param == "staged":
        monkeypatch.setenv("MPSM_DENSE_FLAT", "0")
    else:
        monkeypatch.delenv("MPSM_DENSE_FLAT", raising=False)
    return request.param


def _pack(keys, pays, lower, w):
    pw = 64 - w
    return ((keys - np.uint64(lower)) << np.uint64(pw)) | pays


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(DEV).view(torch.uint64)


def _expect(priv, pub, swap=False):
    """per pair: (count, best, checksum, start, probes, end, examined)"""
    out = []
    for rk, rp in priv:
        for sk, sp in pub:
            if rk.size == 0 or sk.size == 0:
                out.append((0, 0, 0, 0, 0, 0, 0))
                continue
            start, probes = orc.interp_lower_bound(sk, int(rk[0]))
            end = int(np.searchsorted(sk, rk[-1], side="right"))
            cnt, best, examined, _, cs = orc.merge_join_run(rk, rp, sk, sp, start, swap=swap)
            out.append((cnt, best if cnt else 0, cs, start, probes, end, examined))
    return out


def _run(priv, pub, lower, w, swap=False):
    pr = [_dev(_pack(k, p, lower, w)) for k, p in priv]
    pu = [_dev(_pack(k, p, lower, w)) for k, p in pub]
    rec = D.join_pairs_packed(pr, pu, w, lower, swap, _lib.MODE_COUNT)
    return rec.cpu().view(torch.int64).numpy().view(np.uint64).reshape(len(priv) * len(pub), _lib.PAIR_FIELDS)


def _check(priv, pub, lower, w, swap=False):
    rec = _run(priv, pub, lower, w, swap)
    want = _expect(priv, pub, swap)
    cols = [_lib.PAIR_COUNT, _lib.PAIR_BEST, _lib.PAIR_CHECKSUM, _lib.PAIR_START, _lib.PAIR_PROBES, _lib.PAIR_END,
            _lib.PAIR_EXAMINED]
    for p, wnt in enumerate(want):
        got = tuple(int(rec[p, c]) for c in cols)
        if got[0] == 0:
            got = (0, 0, 0) + got[3:]
        assert got == wnt, (p, got, wnt)
        assert int(rec[p, _lib.PAIR_FLAGS]) == 0, p
    return rec


def _fk(n_r, n_s, t_priv, t_pub, seed, lower=1, w=27, pay_bits=32, beyond=0.0):
    """dense R = lower .. lower + n_r - 1 cut into t_priv key ranges; S
    foreign keys (a fraction beyond R's range) in t_pub sorted chunks"""
    rng = np.random.default_rng(seed)
    rk = np.arange(lower, lower + n_r, dtype=np.uint64)
    rp = rng.integers(0, 1 << pay_bits, n_r, dtype=np.uint64)
    hi = lower + int(n_r * (1 + beyond))
    sk = rng.integers(lower, min(hi, lower + (1 << w) - 1), n_s, dtype=np.uint64)
    sp = rng.integers(0, 1 << pay_bits, n_s, dtype=np.uint64)
    cuts = np.linspace(0, n_r, t_priv + 1).astype(np.int64)
    priv = [(rk[a:b], rp[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    pub = []
    for c in np.array_split(np.arange(n_s), t_pub):
        o = np.argsort(sk[c], kind="stable")
        pub.append((sk[c][o], sp[c][o]))
    return priv, pub


@pytest.mark.parametrize("t", [1, 3, 16])
@pytest.mark.parametrize("swap", [False, True])
def test_dense_fk_pairs_match_reference(t, swap):
    priv, pub = _fk(300_000, 1_200_000, t, t, seed=t, beyond=0.2)
    _check(priv, pub, 1, 27, swap)


def test_dense_keys_wider_than_32_bits():
    # w = 40: 64-bit key arithmetic on the dense path (payloads below 2^24)
    priv, pub = _fk(200_000, 700_000, 4, 4, seed=2, lower=(1 << 39) - 100_000, w=40, pay_bits=24)
    _check(priv, pub, (1 << 39) - 100_000, 40)


@pytest.mark.parametrize("frac_wide", [0.0, 0.01, 1.0])
def test_dense_payloads_above_32_bits(frac_wide):
    # w = 27 leaves 37 payload bits; chunks holding a wide payload take the
    # 64-bit hash
    priv, pub = _fk(250_000, 900_000, 2, 5, seed=7)
    rng = np.random.default_rng(11)
    for _, p in priv + pub:
        big = rng.random(p.size) < frac_wide
        p[big] = rng.integers(1 << 32, 1 << 37, int(big.sum()), dtype=np.uint64)
    _check(priv, pub, 1, 27)


def test_dense_and_sparse_runs_in_one_call():
    # run 0 dense, run 1 with a gap, run 2 with a repeated key, run 3 dense
    priv, pub = _fk(400_000, 1_000_000, 4, 3, seed=5)
    k1, p1 = priv[1]
    priv[1] = (np.delete(k1, 5000), np.delete(p1, 5000))
    k2, p2 = priv[2]
    k2 = k2.copy()
    k2[777] = k2[776]
    priv[2] = (k2, p2)
    _check(priv, pub, 1, 27)


def test_overlapping_private_runs_and_edge_sizes():
    # B-MPSM-like private runs over the same keys, a one-tuple run, an empty
    # public run, S keys below and above every run
    rng = np.random.default_rng(9)
    rk = np.arange(1000, 61000, dtype=np.uint64)
    priv = [(rk, rng.integers(0, 1 << 30, rk.size, dtype=np.uint64)),
            (rk[:10_000].copy(), rng.integers(0, 1 << 30, 10_000, dtype=np.uint64)),
            (np.array([5000], np.uint64), np.array([7], np.uint64))]
    sk = np.sort(rng.integers(0, 70_000, 300_000, dtype=np.uint64))
    pub = [(sk, rng.integers(0, 1 << 30, sk.size, dtype=np.uint64)),
           (np.zeros(0, np.uint64), np.zeros(0, np.uint64)),
           (sk[::7].copy(), rng.integers(0, 1 << 30, sk[::7].size, dtype=np.uint64))]
    _check(priv, pub, 0, 27)


def test_dense_heavy_hitter_spans_many_tiles():
    # one key carries 300k S tuples: its block splits into many tiles
    priv, pub = _fk(100_000, 200_000, 1, 2, seed=4)
    k, p = pub[0]
    hot = np.full(300_000, 4242, np.uint64)
    ks = np.concatenate([k, hot])
    ps = np.concatenate([p, np.arange(300_000, dtype=np.uint64)])
    o = np.argsort(ks, kind="stable")
    pub[0] = (ks[o], ps[o])
    _check(priv, pub, 1, 27)


def test_dense_path_flags_unsorted_public_run():
    priv, pub = _fk(100_000, 400_000, 2, 2, seed=8)
    k, p = pub[1]
    k = k.copy()
    i = k.size // 2
    k[i], k[i + 1000] = k[i + 1000], k[i]
    pub[1] = (k, p)
    rec = _run(priv, pub, 1, 27)
    flags = rec[:, _lib.PAIR_FLAGS].astype(np.int64)
    assert flags.reshape(2, 2)[:, 1].any() and (flags & _lib.FLAG_UNSORTED).any()
    assert not flags.reshape(2, 2)[:, 0].any()


@pytest.mark.parametrize("kind", ["dense", "hole", "dup", "random"])
def test_sort_density_probe_and_join_hint(kind):
    """mpsm_sort_packed_dense reports min/max of key - position over its
    output (equal iff the sorted run is dense); the join with that hint gives
    the same records as without it, and a private run changed after its sort
    is flagged by the dense join's key check, never miscounted"""
    rng = np.random.default_rng(5)
    n_r, n_s, lower, w = 50_000, 200_000, 1, 27
    rk = np.arange(lower, lower + n_r, dtype=np.uint64)
    if kind == "hole":
        rk[123] = rk[124]  # one key doubled, one missing
    elif kind == "dup":
        rk[-1] = rk[-2]
    elif kind == "random":
        rk = rng.integers(lower, lower + 4 * n_r, n_r, dtype=np.uint64)
    rk = rk[rng.permutation(n_r)]
    rp = rng.integers(0, 1 << 32, n_r, dtype=np.uint64)
    sk = rng.integers(lower, lower + n_r, n_s, dtype=np.uint64)
    sp = rng.integers(0, 1 << 32, n_s, dtype=np.uint64)

    def sorted_records(k, p, dense=None):
        out, tmp = (torch.empty(k.shape[0], dtype=torch.uint64, device=DEV) for _ in range(2))
        ovf = torch.zeros(1, dtype=torch.int32, device=DEV)
        D.sort_packed(_dev(k), _dev(p), lower, (1 << w) - 1, w, out, tmp, None, ovf, dense)
        return out

    dense = torch.empty(2, dtype=torch.uint32, device=DEV)
    R = sorted_records(rk, rp, dense)
    S = sorted_records(sk, sp)
    d = dense.cpu().numpy()
    assert (d[0] == d[1]) == (kind == "dense"), (kind, d)
    if kind == "dense":
        assert int(d[0]) == 0  # key(R[0]) - lower
    plain = D.join_pairs_packed([R], [S], w, lower, False, _lib.MODE_COUNT)
    hinted = D.join_pairs_packed([R], [S], w, lower, False, _lib.MODE_COUNT, hint=(dense, R))
    assert torch.equal(plain, hinted)
    assert int(hinted[0, _lib.PAIR_FLAGS].item()) == 0
    if kind == "dense":
        o = R.view(torch.int64)
        a = o[1000].clone()
        o[1000] = o[2000]
        o[2000] = a  # after the sort: the probe still says dense
        bad = D.join_pairs_packed([R], [S], w, lower, False, _lib.MODE_COUNT, hint=(dense, R))
        assert int(bad[0, _lib.PAIR_FLAGS].item()) & _lib.FLAG_UNSORTED
