import time, sys, json
sys.path.insert(0, '.')
import torch, synth
from paper_1908_00213_b200 import Comm, cmn
lib = cmn.lib()
shapes = synth.mlp_shapes()
comm = Comm.init(0, 1, 0)
w = [torch.from_numpy(p).cuda() for p in synth.params(shapes)]
comm.register_params(w)
g = comm.prepare([torch.from_numpy(x).cuda() for x in synth.grads(shapes, workers=1)[0]])
s = torch.cuda.current_stream().cuda_stream
def t(fn, n=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(n): fn()
    b = time.perf_counter()
    torch.cuda.synchronize()
    return (b - a) / n * 1e6
h = comm._h
res = {
 "ctypes_cmn_version": t(lambda: lib.cmn_version()),
 "torch_current_stream": t(lambda: torch.cuda.current_stream().cuda_stream),
 "raw_ctypes_cmn_step": t(lambda: lib.cmn_step(h, g.arr, 0, 0.1, 0.9, s)),
 "binding_step_explicit_stream": t(lambda: comm.step(g, "fp32", 0.1, 0.9, s)),
 "binding_step_default_stream": t(lambda: comm.step(g, "fp32", 0.1, 0.9)),
 "torch_small_add_": t(lambda: w[5].add_(0.0)),
}
print(json.dumps(res))
