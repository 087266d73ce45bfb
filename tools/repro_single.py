import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_04936_b200 as lg
ds = lg.generate_dataset(500, 12, 3, seed=0)
idx = lg.build(ds)
qs = lg.generate_queries(ds, 120, seed=1)
for rep in range(3):
    for i, q in enumerate(qs):
        k = (1, 5, 50)[i % 3]
        for mode in ("strict", "complete"):
            r = idx.query(q, k, mode)
    print("rep", rep, "ok", flush=True)
