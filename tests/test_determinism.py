"""Cross-process, cross-launch-geometry determinism (north star: "identical
across repeated runs"; reference acceptance C2, pkg/tests/test_acceptance.py:94-119).

Ten subprocesses (PYTHONHASHSEED varied, as the reference varies it) each
build the index from scratch and run every query path several times; all
digests must be identical.  Some runs also change the launch geometry the
host picks — full-scan chunk count (which changes the cross-chunk pruning
hint's timing and the merge fan-in) and the warps per query CTA — so results
are proven independent of grid sizes and of the SM count of the box.
One run's results are additionally checked against the C oracle in-process
by tests/test_gpu_configs.py (same generator, same paths).
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "tests", "determinism_gpu_driver.py")

GEOMETRIES = [
    {},
    {"LCP_FULLSCAN_CHUNKS": "1"},
    {"LCP_FULLSCAN_CHUNKS": "7"},
    {"LCP_FULLSCAN_CHUNKS": "257"},
    {"LCP_WPC_MIN": "32"},
    {"LCP_WPC_MIN": "4", "LCP_FULLSCAN_CHUNKS": "64"},
    {"LCP_NO_GRAPH_CACHE": "1"},
    {},
    {"LCP_FULLSCAN_CHUNKS": "3"},
    {},
]


@pytest.mark.gpu
def test_cross_process_determinism(gpu):
    digests = []
    for i, extra in enumerate(GEOMETRIES):
        env = dict(os.environ)
        env["PYTHONHASHSEED"] = str(1000 + 17 * i)
        env.update(extra)
        r = subprocess.run([sys.executable, DRIVER, "60000", "24", "4", "11", "2"], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        lines = r.stdout.split()
        assert len(lines) == 2 and lines[0] == lines[1], (extra, lines)  # repeated in-process
        digests.append((extra, lines[0]))
    assert len({d for _, d in digests}) == 1, digests
