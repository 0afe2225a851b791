"""Host-side pieces around the hot path, on CPU: the instance-file reader
(read_instances, proj/src/data.cpp:72-110) against the compiled reference on
the same files (values and error messages), and the ledger arithmetic
(kstep_ratio, proj/src/ledger.cpp:132-145) against the reference's own
closed-form checks (proj/tests/test_ledger.cpp:50-86)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2201_05500_b200 as kp
from oracle import oracle as O
from paper_2201_05500_b200.data import make_batch

GOOD = [
    "1\t5,3,5\n0\t7\n",                       # duplicates, unsorted
    "\n1\t1,2,3\n\n0\t4\n",                    # empty lines skipped
    "1\t3,,4,\n",                              # empty tokens skipped
    "0\t 7,+8,9\n",                            # stoull: leading blank, sign
    "1\t-1\n",                                 # stoull("-1") wraps to u64 max
    "1\t12abc,18446744073709551615\n",         # trailing junk ignored; u64 max
    "0\t0\n1\t0,0,0\n",
]
BAD = [
    ("1 5,6\n", "line 1: missing tab separator"),
    ("2\t5\n", "line 1: label must be 0 or 1"),
    ("1\t5\n0\tabc\n", "line 2: bad feature id 'abc'"),
    ("1\t18446744073709551616\n", "bad feature id '18446744073709551616'"),
    ("1\t\n", "line 1: no feature ids"),
    ("1\t,,\n", "line 1: no feature ids"),
    (" 1\t5\n", "label must be 0 or 1"),
]


def _ref_ok():
    return O.ref_available()


@pytest.mark.parametrize("text", GOOD)
def test_read_instances_matches_reference(tmp_path, text):
    f = tmp_path / "in.tsv"
    f.write_text(text)
    offs, keys, labels = kp.read_instances(str(f))
    if _ref_ok():
        ro, rk, rl = O.ref_read_instances(f)
        assert np.array_equal(offs.astype(np.uint64), ro)
        assert np.array_equal(keys, rk) and np.array_equal(labels, rl)
    for i in range(len(labels)):  # each instance ascending + deduped
        k = keys[offs[i]:offs[i + 1]]
        assert len(k) and np.all(np.diff(k.astype(np.float64)) > 0) or len(k) == 1


@pytest.mark.parametrize("text,msg", BAD)
def test_read_instances_errors_match_reference(tmp_path, text, msg):
    f = tmp_path / "bad.tsv"
    f.write_text(text)
    with pytest.raises(kp.KpsimError) as e:
        kp.read_instances(str(f))
    assert msg in str(e.value)
    if _ref_ok():
        with pytest.raises(RuntimeError) as r:
            O.ref_read_instances(f)
        assert str(r.value) == str(e.value)


def test_read_instances_missing_file(tmp_path):
    with pytest.raises(kp.KpsimError, match="cannot open instance file"):
        kp.read_instances(str(tmp_path / "nope.tsv"))


def test_write_read_round_trip_and_reference(tmp_path):
    """write_instances -> read_instances is the identity on a folded Zipf
    batch, and the reference reads our file to the same CSR."""
    bt = make_batch(2000, V=10**8, zipf_s=1.1, n_slots=26, seed=3).folded()
    f = tmp_path / "b.tsv"
    kp.write_instances(str(f), bt.offs, bt.keys, bt.labels)
    offs, keys, labels = kp.read_instances(str(f))
    assert np.array_equal(offs, bt.offs) and np.array_equal(keys, bt.keys)
    assert np.array_equal(labels, bt.labels)
    if _ref_ok():
        ro, rk, rl = O.ref_read_instances(f)
        assert np.array_equal(ro, offs.astype(np.uint64)) and np.array_equal(rk, keys)


def _sched(T, k, N, D, S):
    """schedule_ledger (ledger.cpp:161-180) as a ledger dict"""
    dense = (T // k) * N
    sparse = T * N if S else 0
    return {"dense_merge": {"bytes": dense * D, "count": dense},
            "sparse_sync": {"bytes": sparse * S, "count": sparse}}


def test_kstep_ratio_reference_checks():
    """proj/tests/test_ledger.cpp:50-86 restated: dense ratio floor(T/k)/T,
    total (0.1 D + S)/(D + S) = 0.82 at S = 4D, monotone in k, zero-byte
    baseline is an error."""
    T, N, D, S = 1000, 4, 4096, 4 * 4096
    base = _sched(T, 1, N, D, S)
    for k in (10, 20, 50, 100):
        r = kp.kstep_ratio(_sched(T, k, N, D, S), base)
        assert r["dense_bytes"] == pytest.approx((T // k) / T, rel=1e-15)
    assert kp.kstep_ratio(_sched(T, 10, N, D, S), base)["total_bytes"] == pytest.approx(0.82, rel=1e-13)
    prev = 2.0
    for k in (10, 20, 50, 100, 200):
        r = kp.kstep_ratio(_sched(T, k, N, D, S), base)["total_bytes"]
        assert r < prev
        prev = r
    with pytest.raises(kp.KpsimError, match="zero-byte baseline"):
        kp.kstep_ratio(base, {})
