import faulthandler, sys, threading, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
faulthandler.dump_traceback_later(40, exit=True)
import paper_2505_22296_b200 as P
fab = P.Fabric(2)
def body(r):
    print("rank", r, "start", flush=True)
    n = P.all_reduce_count((fab, r), 3 + r)
    print("rank", r, "count", n, flush=True)
    v = P.losses._group((fab, r)).values([1.0 + r])
    print("rank", r, "values", v, flush=True)
    x = torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda")
    s = P.logprob_sum_allreduce((fab, r), x)
    print("rank", r, "sum", s.item(), flush=True)
th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
[t.start() for t in th]; [t.join() for t in th]
print("done")
