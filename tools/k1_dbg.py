import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2310_19295_b200 import graphgen as gg, evaluator as ev
from paper_2310_19295_b200.graph import load_graph
from oracle import coracle
g = load_graph(gg.config_doc("gpt2-small"))
for B in (64, 300, 2000, 16384):
    orders = ev.generate_orders(g, 0, 0, B)
    host = orders.cpu().numpy()
    want = coracle.eval_orders(coracle.CGraph(g), host[:min(B,2000)])
    p, a, v = (x.cpu().numpy() for x in ev.evaluate_orders(g, orders))
    m = min(B, 2000)
    bad = np.nonzero((v[:m] != want[2]) | (p[:m] != want[0]))[0]
    print("B", B, "mismatches", len(bad), bad[:20].tolist(), "valid", v[:m].sum(), want[2].sum())
