"""NEXT f4: the committed measured batch WCET table (profiles/r1_batch_wcet_tables.json,
written on a B200 by tools/batch_wcet_tables.py) has SPEC.md's BatchWcetTables form
and its invariants: batching property C_B(n) <= n C(1) (§IV-A "C_{B^S} <= Σ
C_i^S") on the 99th-percentile times, and monotone in level and in n on the means (S:55,
within 1 % timing noise)."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH = os.path.join(ROOT, "profiles", "r1_batch_wcet_tables.json")


@pytest.fixture(scope="module")
def table():
    with open(PATH) as f:
        return json.load(f)


def test_form(table):
    assert set(table["levels"]) == {"S", "M", "L"}
    ks = [table["levels"][w]["k"] for w in ("S", "M", "L")]
    assert ks == sorted(ks) and ks[-1] == 400
    n_max = len(table["coarse"])
    assert [int(n) for n in table["coarse"]] == list(range(1, n_max + 1))
    for w in ("S", "M", "L"):
        assert [int(n) for n in table["fine"][w]] == list(range(1, n_max + 1))
    for e in [*table["coarse"].values(), *(v for w in table["fine"].values() for v in w.values())]:
        assert 0 < e["mean_ms"] <= e["wcet_ms"] and e["p99_ms"] <= e["wcet_ms"] and e["runs"] >= 300


def test_batching_property(table):
    c = table["coarse"]
    assert all(c[n]["p99_ms"] <= int(n) * c["1"]["p99_ms"] for n in c)
    for w, f in table["fine"].items():
        assert all(f[n]["p99_ms"] <= int(n) * f["1"]["p99_ms"] for n in f), w


def test_monotone_in_level_and_n(table):
    f = table["fine"]
    n_max = len(table["coarse"])
    for n in map(str, range(1, n_max + 1)):
        assert f["S"][n]["mean_ms"] <= 1.01 * f["M"][n]["mean_ms"] <= 1.01 ** 2 * f["L"][n]["mean_ms"]
    for w in f:
        for n in range(1, n_max):
            assert f[w][str(n)]["mean_ms"] <= 1.01 * f[w][str(n + 1)]["mean_ms"], (w, n)
