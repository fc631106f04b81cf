import sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from conftest import golden
from paper_2310_19295_b200.graph import load_graph
from paper_2310_19295_b200.evaluator import evaluate_orders, device_graph
for idx, e in enumerate(golden("peaks")["small_dags"]):
    g = load_graph(e["doc"]); n = len(g.ops)
    rows = [r for r in e["rows"] if len(r["order"]) == n]
    o = np.array([r["order"] for r in rows], np.int64).reshape(len(rows), n)
    print(idx, n, device_graph(g).info(), o.shape, flush=True)
    evaluate_orders(g, o)
print("ok")
