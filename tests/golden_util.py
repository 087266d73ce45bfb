"""Helpers to regenerate golden-case inputs and read expected outputs."""

from __future__ import annotations

import hashlib

import numpy as np

from paper_2602_04936_b200.datagen import generate_dataset


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_dataset(case):
    ds = generate_dataset(case["n"], case["length"], case["sigma"], seed=case["seed"],
                          distribution=case["distribution"])
    assert sha(ds.items) == case["dataset_sha256"], f"datagen drifted for {case['name']}"
    return ds


def expected_rows(arrays, prefix, i):
    h = int(arrays[prefix + "hits"][i])
    return list(zip(arrays[prefix + "ids"][i, :h].tolist(), arrays[prefix + "lcps"][i, :h].tolist()))
