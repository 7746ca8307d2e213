"""Where the one-shot C-ABI call spends its time (cfg4): host analysis, upload,
kernel, D2H into pinned memory."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_04285_b200 import engine as E, graph as G, models as M, abi

g, t = M.cfg4()
f = G.flatten(g)
lib = abi.load_engine()
gd, td = f.desc(), t.desc()
def now():
    torch.cuda.synchronize()
    return time.perf_counter()
for rep in range(6):
    t0 = now()
    plan = E.Plan(f, t, device=0)
    t1 = now()
    plan.upload(0)
    t2 = now()
    ne, nn = plan.sizes["num_aux_edges"], plan.sizes["num_aux_nodes"]
    host = {k: torch.empty(ne, dtype=torch.float64, pin_memory=True).numpy()
            for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
    host.update({k: torch.empty(nn, dtype=torch.float64, pin_memory=True).numpy()
                 for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes")})
    class H: pass
    hv = H()
    for k, v in host.items(): setattr(hv, k, v)
    hv.records = hv.row_min_cost_s = hv.row_min_volume_bytes = None
    hs = E.cost_struct(hv)
    t3 = now()
    o = abi.tp_build_opts(0, -1, 0, 0, None)
    st = lib.tp_plan_execute_host(plan.handle, C.byref(o), None, C.byref(hs))
    t4 = now()
    o2 = abi.tp_build_opts(0, -1, 0, 0, None)
    t5 = now()
    st = lib.tp_build_cost_tensors(C.byref(gd), C.byref(td), C.byref(o2), None, C.byref(hs))
    t6 = now()
    print(f"create {1e3*(t1-t0):.3f} ms, upload {1e3*(t2-t1):.3f} ms, execute_host (kernel + D2H 53.7 MB) {1e3*(t4-t3):.3f} ms, one-shot total {1e3*(t6-t5):.3f} ms")
    del plan
