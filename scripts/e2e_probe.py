import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch, ctypes as C
import paper_2309_10212_b200 as wc
from paper_2309_10212_b200.benchmark import orbit_camera
wc._lib.ensure_device(0)
f = wc.volume.separable_field("turbulence", (2048, 2048, 1920), 1)
cv = wc.compress_separable(f, 16); g = wc.build_grids(cv)
r = cv.raw_block_ranges; lo, hi = float(r[:,0].min()), float(r[:,1].max()); iso = lo + 0.5*(hi-lo)
cam = orbit_camera(cv.dims, 0, 1)
opts = wc.RenderOptions(width=1920, height=1080)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for i in range(12):
    if i >= 6: flush.zero_()
    torch.cuda.synchronize(); t=time.perf_counter()
    fb, st = wc.render(cv, g, cam, iso, opts)
    t1=time.perf_counter()
    s = wc.engine.session_pool.items[-1][1]
    print('render wall %.3f ms  frame %.3f ms  passes %d' % ((t1-t)*1e3, s.frame_ms(), len(st)))
base = wc._lib.pinned_pool.get(8*s.n)
attr = C.c_int*8
from ctypes import byref
# check pinned via torch? use cudart
cudart = C.CDLL("libcudart.so")
class Attr(C.Structure):
    _fields_=[("type",C.c_int),("device",C.c_int),("devicePointer",C.c_void_p),("hostPointer",C.c_void_p)]
a=Attr(); rc=cudart.cudaPointerGetAttributes(C.byref(a), C.c_void_p(base.ctypes.data)); print('ptr attr rc', rc, 'type', a.type)
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    st = s.render_frame(cam, iso)
    t1=time.perf_counter(); rgba, depth = s.read(); t2=time.perf_counter()
    print('render_frame %.3f ms read %.3f ms' % ((t1-t)*1e3, (t2-t1)*1e3))
