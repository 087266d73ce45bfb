"""Golden scenario reports from the reference's own runner.

Run in a container that has /root/reference (read-only):

    python tests/golden/make_golden_scenarios.py

Executes ``lcpsearch.run_scenario`` (pkg/src/lcpsearch/bench.py:470-472) on
small configs and stores each report's deterministic sections (``config`` and
``results``; ``wall_clock`` varies by design) in scenarios_v1.json.
"""

from __future__ import annotations

import json
import os
import sys

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

CONFIGS = [
    # the reference tests' toy config (pkg/tests/test_bench.py:96-107)
    dict(scenario="sustained", seed=42, n_items=400, seq_len=10, alphabet=2, k=5, query_count=60),
    dict(scenario="sustained", seed=42, n_items=400, seq_len=10, alphabet=2, k=5, query_count=60, workers=4),
    dict(scenario="sustained", seed=7, n_items=3000, seq_len=16, alphabet=4, k=10, query_count=500,
         mode="strict"),
    dict(scenario="sustained", seed=8, n_items=5000, seq_len=24, alphabet=4, k=10, query_count=700,
         prefix_len=12, distribution="clustered"),
    dict(scenario="gnc", seed=42, n_items=400, seq_len=10, alphabet=2, k=5, query_count=60, steps=50),
    dict(scenario="gnc", seed=4, n_items=10000, seq_len=24, alphabet=4, k=5, steps=300, prefix_len=12),
    dict(scenario="tal_sweep", seed=42, n_items=4096, seq_len=16, alphabet=2, k=5, query_count=60,
         bucket_counts=(1, 4, 16)),
    dict(scenario="tal_sweep", seed=9, n_items=6000, seq_len=12, alphabet=4, k=10, query_count=200,
         bucket_counts=(1, 4, 16, 64, 256)),
    dict(scenario="memo", seed=42, n_items=400, seq_len=10, alphabet=2, k=5, query_count=60),
    dict(scenario="memo", seed=5, n_items=2000, seq_len=6, alphabet=2, k=7, query_count=300),
]


def main() -> int:
    sys.path.insert(0, REF_SRC)
    import lcpsearch as ref  # noqa: E402

    # a reference snapshot, served by the sustained scenario through index_path
    snap = os.path.join(HERE, "snap_scenario.lcpi")
    import lcpsearch.storage  # noqa: E402,F401

    ref.storage.write_index(snap, ref.build(ref.generate_dataset(1000, 10, 4, seed=21)))
    configs = CONFIGS + [dict(scenario="sustained", seed=22, seq_len=10, alphabet=4, k=10, query_count=400,
                              index_path="tests/golden/snap_scenario.lcpi")]
    out = []
    cwd = os.getcwd()
    os.chdir(os.path.dirname(os.path.dirname(HERE)))  # index_path is relative to the repo root
    for cfg in configs:
        rep = ref.run_scenario(ref.ScenarioConfig(**cfg)).to_machine()
        out.append({"args": {k: (list(v) if isinstance(v, tuple) else v) for k, v in cfg.items()},
                    "config": rep["config"], "results": rep["results"],
                    "schema_version": rep["schema_version"]})
    os.chdir(cwd)
    with open(os.path.join(HERE, "scenarios_v1.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_scenarios.py", "reference": REF_SRC,
                   "reports": out}, f, indent=1, sort_keys=True)
    print(f"wrote {len(out)} scenario reports")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
