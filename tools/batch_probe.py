"""Config 5a on one GPU: n independent 513^3 fp32 fields in flight, each on
its own stream / context / captured step graph, free-running (no per-step
join): aggregate decompose+recompose GB/s of input."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_05872_b200 as mg
from synthetic_fields import config2_field

DIMS = (513, 513, 513)


def measure(inflight, steps=10, join_each=False):
    dev = torch.device("cuda", 0)
    h = mg.GridHierarchy.create(DIMS)
    fields = [config2_field(DIMS, seed=1000 + i, device=dev) for i in range(inflight)]
    streams = [torch.cuda.Stream(dev) for _ in fields]
    graphs, ctxs = [], []
    for f, st in zip(fields, streams):
        ws = mg.SolverWorkspace(device=0)
        ctxs.append(ws)
        st.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(st):
            mg.recompose(mg.decompose(f, h, 0, ws), ws)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                mg.recompose(mg.decompose(f, h, 0, ws), ws)
        graphs.append(g)
    torch.cuda.synchronize()
    main = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run(k):
        if join_each:
            for _ in range(k):
                for g, st in zip(graphs, streams):
                    st.wait_stream(main)
                    with torch.cuda.stream(st):
                        g.replay()
                for st in streams:
                    main.wait_stream(st)
        else:
            for st in streams:
                st.wait_stream(main)
            for _ in range(k):
                for g, st in zip(graphs, streams):
                    with torch.cuda.stream(st):
                        g.replay()
            for st in streams:
                main.wait_stream(st)

    run(2)
    torch.cuda.synchronize()
    e0.record(main)
    run(steps)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    nbytes = sum(f.numel() * f.element_size() for f in fields)
    return ms, nbytes / (ms * 1e-3) / 1e9


if __name__ == "__main__":
    for n in (1, 2, 3, 4, 6, 8):
        for je in (True, False):
            ms, gbs = measure(n, join_each=je)
            print(f"in flight {n} join_each {je}: {ms:.3f} ms per round, {gbs:.1f} GB/s of input", flush=True)
