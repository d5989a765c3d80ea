"""NEXT f4: the committed measured batch WCET table (profiles/r2_batch_wcet_tables.json, written
on a B200 by tools/batch_wcet_tables.py) has SPEC.md's BatchWcetTables form, and the
invariants S:52-55 hold EXACTLY on the Duration it publishes (wcet_ms): the batching property
coarse(n) <= n coarse(1), fine(w,n) <= n fine(w,1) (§IV-A "C_{B^S} <= sum C_i^S"), and
fine(., n) non-decreasing in level and in n.  wcet_ms is the measured 99th percentile raised to
its monotone envelope (a WCET bound may only be raised); the observed maxima are max_ms."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH = os.path.join(ROOT, "profiles", "r2_batch_wcet_tables.json")
LEVELS = ("S", "M", "L")


@pytest.fixture(scope="module")
def table():
    with open(PATH) as f:
        return json.load(f)


def test_form(table):
    assert set(table["levels"]) == set(LEVELS)
    ks = [table["levels"][w]["k"] for w in LEVELS]
    assert ks == sorted(ks) and ks[-1] == 400
    n_max = len(table["coarse"])
    assert [int(n) for n in table["coarse"]] == list(range(1, n_max + 1))
    for w in LEVELS:
        assert [int(n) for n in table["fine"][w]] == list(range(1, n_max + 1))
    for e in [*table["coarse"].values(), *(v for w in table["fine"].values() for v in w.values())]:
        assert 0 < e["mean_ms"] <= e["p99_ms"] <= e["max_ms"] and e["p99_ms"] <= e["wcet_ms"] and e["runs"] >= 300


def test_published_wcet_is_the_monotone_envelope_of_p99(table):
    c, f = table["coarse"], table["fine"]
    n_max = len(c)
    for n in range(1, n_max + 1):
        assert c[str(n)]["wcet_ms"] == max(c[str(i)]["p99_ms"] for i in range(1, n + 1))
        for li, w in enumerate(LEVELS):
            env = max(f[v][str(i)]["p99_ms"] for v in LEVELS[:li + 1] for i in range(1, n + 1))
            assert f[w][str(n)]["wcet_ms"] == pytest.approx(env, abs=1e-4)


def test_batching_property_on_wcet(table):
    c = table["coarse"]
    assert all(c[n]["wcet_ms"] <= int(n) * c["1"]["wcet_ms"] for n in c)
    for w, f in table["fine"].items():
        assert all(f[n]["wcet_ms"] <= int(n) * f["1"]["wcet_ms"] for n in f), w


def test_monotone_in_level_and_n_on_wcet(table):
    f = table["fine"]
    n_max = len(table["coarse"])
    for n in map(str, range(1, n_max + 1)):
        assert f["S"][n]["wcet_ms"] <= f["M"][n]["wcet_ms"] <= f["L"][n]["wcet_ms"]
    for w in f:
        for n in range(1, n_max):
            assert f[w][str(n)]["wcet_ms"] <= f[w][str(n + 1)]["wcet_ms"], (w, n)
    assert all(table["invariants"].values())
