"""Benchmark scenarios on the GPU backend (reference: pkg/tests/test_bench.py).

CPU: latency statistics, the memory wall and config validation.  GPU: every
golden report from the reference's own runner (tests/golden/scenarios_v1.json)
must have byte-for-byte equal ``config`` and ``results`` sections here, plus
the reference test suite's scenario invariants.
"""

import json
import math
import os

import pytest

from paper_2602_04936_b200 import ConfigError, ScenarioConfig, memory_wall, run_scenario
from paper_2602_04936_b200.scenarios import GIB, LatencyStats, ScenarioReport, format_byte_size

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "scenarios_v1.json")))["reports"]


# ------------------------------------------------------------------ CPU
def test_percentiles_are_nearest_rank():
    stats = LatencyStats.from_samples([i / 1000 for i in range(1, 101)], elapsed_s=1.0)
    assert stats.p50 == pytest.approx(0.050) and stats.p95 == pytest.approx(0.095)
    assert stats.p99 == pytest.approx(0.099) and stats.qps == pytest.approx(100.0)
    assert LatencyStats.from_samples([], elapsed_s=1.0).total_queries == 0


@pytest.mark.parametrize("n,display,feasible", [(100_000, "18.63 GiB", True), (200_000, "74.51 GiB", True),
                                                (500_000, "465.66 GiB", False), (1_000_000, "1.86 TiB", False)])
def test_memory_wall_reference_rows(n, display, feasible):
    est = memory_wall(n, budget_bytes=80 * GIB)
    assert est.materialization_bytes == n * n * 2
    assert est.materialization_display == display and est.feasible is feasible


def test_memory_wall_misc():
    assert format_byte_size(2_000_000 * 2_000_000 * 2) == "7.45 TiB"
    assert memory_wall(100_000, index_bytes=68_400_000).ratio == pytest.approx(20_000_000_000 / 68_400_000)
    with pytest.raises(ConfigError):
        memory_wall(0)


def test_config_validation():
    with pytest.raises(ConfigError):
        ScenarioConfig(scenario="warp", seed=1)
    for bad in (dict(n_items=0), dict(mode="fast"), dict(duration_s=-2.0), dict(bucket_counts=(1, 0)),
                dict(index_path="x.lcpi", prefix_len=3), dict(seed=None)):
        with pytest.raises(ConfigError):
            ScenarioConfig(**{"scenario": "sustained", "seed": 1, **bad})
    for g in GOLDEN:  # the config section is a pure function of the arguments
        assert ScenarioConfig(**g["args"]).as_dict() == g["config"]


def test_text_rendering_matches_reference_format():
    rep = ScenarioReport("sustained", {"seed": 42}, {"work": {"queries": 3}, "x": 0.5},
                         {"sweep": [{"a": 1}], "l": [2, 3]})
    text = rep.to_text()
    assert text.splitlines()[:3] == ["lcpsearch scenario report", "schema: 1", "scenario: sustained"]
    for line in ("[config]", "seed: 42", "work.queries: 3", "x: 0.5", "sweep.0.a: 1", "l.1: 3"):
        assert line in text
    assert json.loads(rep.to_json())["schema_version"] == "1"


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(GOLDEN)))
def test_results_equal_reference_runner(gpu, i, monkeypatch):
    g = GOLDEN[i]
    monkeypatch.chdir(os.path.dirname(HERE))  # index_path cases are relative to the repo root
    rep = json.loads(json.dumps(run_scenario(ScenarioConfig(**g["args"])).to_machine()))
    assert rep["schema_version"] == g["schema_version"]
    assert rep["config"] == g["config"]
    assert rep["results"] == g["results"]


@pytest.mark.gpu
def test_scenario_invariants(gpu, tmp_path):
    from paper_2602_04936_b200 import InvalidStateError

    toy = dict(seed=42, n_items=400, seq_len=10, alphabet=2, k=5, query_count=60)
    m = run_scenario(ScenarioConfig(scenario="sustained", **toy)).to_machine()
    lat = m["wall_clock"]["latency"]
    assert lat["p50_ms"] <= lat["p95_ms"] <= lat["p99_ms"] and lat["total_queries"] == 60
    g = run_scenario(ScenarioConfig(scenario="gnc", steps=50, **toy)).to_machine()
    assert g["wall_clock"]["steps_per_second"] > 0
    memo = run_scenario(ScenarioConfig(scenario="memo", **toy)).to_machine()
    assert memo["results"]["hot_work"]["cache_hits"] == 60 and memo["wall_clock"]["speedup"] > 0
    tal = run_scenario(ScenarioConfig(scenario="tal_sweep", **{**toy, "n_items": 4096, "seq_len": 16},
                                      bucket_counts=(1, 4, 16))).to_machine()
    red = [r["reduction"] for r in tal["results"]["sweep"]]
    assert red[0] == pytest.approx(1.0) and red == sorted(red)
    d = run_scenario(ScenarioConfig(scenario="sustained", duration_s=0.2, **{**toy, "query_count": 10}))
    d = d.to_machine()
    assert d["wall_clock"]["work"]["queries"] > 0 and d["wall_clock"]["elapsed_s"] >= 0.2
    assert not math.isnan(d["wall_clock"]["latency"]["p50_ms"]) and "work" not in d["results"]
    with pytest.raises(InvalidStateError):
        run_scenario(ScenarioConfig(scenario="sustained", index_path=str(tmp_path / "none.lcpi"), **toy))
    # a snapshot-loaded index serves the sustained scenario with the same results
    from paper_2602_04936_b200 import build, generate_dataset, storage

    path = tmp_path / "idx.lcpi"
    storage.write_index(str(path), build(generate_dataset(400, 10, 2, 42)))
    a = run_scenario(ScenarioConfig(scenario="sustained", index_path=str(path), **toy)).to_machine()
    assert a["results"]["index_nodes"] == m["results"]["index_nodes"]
    assert a["results"]["determinism"]["byte_identical"] is True
