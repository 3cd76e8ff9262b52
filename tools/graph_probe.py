"""CUDA-graph replay vs per-call launches of one solve (launch-bound small grids).

    python tools/graph_probe.py --config c1 --steps 200
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1409_8116_b200 as fp  # noqa: E402
from paper_1409_8116_b200 import _native as nat  # noqa: E402
from paper_1409_8116_b200 import _device as dv  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--steps", type=int, default=200)
a = ap.parse_args()
config, _ = bench.make_config(a.config)
plan = fp.SolverPlan(config)
dev = torch.device("cuda", 0)
tdt = dv.torch_dtype(config.dtype)
rhs = torch.randn(config.shape, dtype=tdt, device=dev)
out = torch.empty_like(rhs)
wsb = plan.workspace_bytes(out_dense=True)
work = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
info = torch.zeros(16, dtype=torch.uint8, device=dev)
rs, os_ = nat.strides_array(rhs.stride()), nat.strides_array(out.stride())
rdt = dv.fp_dtype_of_torch(tdt)


def step():
    sh = torch.cuda.current_stream(dev).cuda_stream
    nat.check(plan._lib.fp_solve_ex(plan._handle, rhs.data_ptr(), rdt, rs, out.data_ptr(), os_, work.data_ptr(),
                                    wsb, sh, info.data_ptr(), None, None))


def timed(fn, k):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


plain = timed(step, a.steps)
ref = out.clone()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
graph = timed(g.replay, a.steps)
same = torch.equal(out, ref)
print(json.dumps({"config": a.config, "per_call_ms": round(plain, 5), "graph_ms": round(graph, 5), "identical": same}))
