import ctypes, json, time, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import _native, configs
L = _native.lib()
def t(fn, reps=20):
    fn(); fn()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    return (time.perf_counter() - t0) / reps * 1e6
res = {}
tiny = sk.Matrix2D.from_array(np.zeros((1, 128), np.float32), pinned=True)
out_t = sk.alloc_matrix(1, 128, pinned=True)
res['py_api_1x128_us'] = t(lambda: sk.softmax(tiny, sk.KernelVariant.REFERENCE_CLIPPED, out=out_t))
bad = ctypes.c_int64(-1)
res['c_host_1x128_us'] = t(lambda: L.sk_softmax_f32_host(tiny.data.ctypes.data, out_t.data.ctypes.data, 1, 128, 0, 0, ctypes.byref(bad)))
spec = configs.get('c2')
m = sk.Matrix2D.from_array(configs.generate(spec), pinned=True)
o = sk.alloc_matrix(spec.rows, spec.cols, pinned=True)
res['py_api_c2_us'] = t(lambda: sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o))
res['c_host_c2_us'] = t(lambda: L.sk_softmax_f32_host(m.data.ctypes.data, o.data.ctypes.data, spec.rows, spec.cols, 0, 0, ctypes.byref(bad)))
# ideal: torch copies, 4 chunks, two streams, no kernel
h = torch.from_numpy(m.data.reshape(-1)); ho = torch.from_numpy(o.data.reshape(-1))
d = torch.empty_like(h, device='cuda'); s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def pipe(n=8):
    cs = h.numel() // n
    evs = []
    for k in range(n):
        with torch.cuda.stream(s1):
            d[k*cs:(k+1)*cs].copy_(h[k*cs:(k+1)*cs], non_blocking=True)
            e = torch.cuda.Event(); e.record(s1)
        s2.wait_event(e)
        with torch.cuda.stream(s2):
            ho[k*cs:(k+1)*cs].copy_(d[k*cs:(k+1)*cs], non_blocking=True)
    torch.cuda.synchronize()
for n in (4, 8, 16):
    res[f'copy_pipe_{n}_us'] = t(lambda: pipe(n))
print(json.dumps(res))
