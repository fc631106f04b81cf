import sys, torch, json
sys.path.insert(0, '/root/repo')
from paper_2310_19295_b200 import evaluator as ev, graphgen as gg
from paper_2310_19295_b200.graph import load_graph
for name in ['gpt2-xl','gpt2-small']:
    g = load_graph(gg.config_doc(name))
    big = ev.generate_orders(g, 0, 0, 65536)
    print(name, 'gen dtype', big.dtype, flush=True)
    for B in (8192, 16384, 32768, 65536):
        for dt in (torch.int32, torch.uint16):
            o = big[:B].to(dt).contiguous()
            ev.evaluate_orders(g, o); torch.cuda.synchronize()
            ts=[]
            for _ in range(5):
                e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
                e0.record(); ev.evaluate_orders(g, o); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            print(json.dumps({"graph":name,"B":B,"dtype":str(dt),"ms":min(ts),"us_per_1k":min(ts)/B*1e6}), flush=True)
