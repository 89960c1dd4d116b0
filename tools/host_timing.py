"""Wall-clock per-view timing of encode_views_device with 1 and 2 lanes (dev tool)."""
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2505_08124_b200._lib import Context
from harness.workload import make_bench_workload
wl = make_bench_workload(2_000_000, 1000, 1152, 864, 64, 512, seed=1, views=list(range(48)))
ctx = Context(0); ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
dev=torch.device('cuda',0)
runs=np.concatenate([m[3] for m in wl.masks]); base=0; offs=[]
for m in wl.masks: offs.append(torch.from_numpy(m[4].astype(np.int64)+base).to(dev)); base+=int(m[4][-1])
d_runs=torch.from_numpy(runs.view(np.int32)).to(dev); clips=[torch.from_numpy(m[5]).to(dev) for m in wl.masks]
dm=[(m[0],m[1],m[2],d_runs.data_ptr(),o.data_ptr(),c.data_ptr(),int(m[4][-1]-m[4][0])) for m,o,c in zip(wl.masks,offs,clips)]
ctx.encode_begin(512); ctx.encode_views_device(wl.cams, dm); torch.cuda.synchronize()
for lanes in (2,1):
    ctx.set_lanes(lanes)
    t=time.perf_counter(); ctx.encode_begin(512); ctx.encode_views_device(wl.cams, dm); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("lanes", lanes, "wall ms/view", dt/48*1e3)
import cProfile
