import os, sys, time, tempfile, json
sys.path.insert(0, '/root/repo')
import torch
from paper_2511_14124_b200 import traces as T
from paper_2511_14124_b200.engine import Engine
wd = tempfile.mkdtemp(dir='/dev/shm')
info = T.config_c2(wd)
e = Engine(info['trace'], info['machine'], {'policy': 'tencache'})
e.seed(0)
st = torch.cuda.current_stream()
kw = dict(lr=1e-4, compute_mode=1, spin_ctas=1, stream=st.cuda_stream)
for _ in range(3): e.iteration(**kw)
e.sync()
ts = []
for k in range(6):
    t0 = time.perf_counter(); e.iteration(last=k == 5, **kw); t1 = time.perf_counter()
    ts.append((t1 - t0) * 1e3)
e.sync()
r = []
for k in range(6):
    t0 = time.perf_counter(); e.iteration(last=k == 5, **kw); t1 = time.perf_counter(); e.step_result(); t2 = time.perf_counter()
    r.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3))
e.sync()
print(json.dumps({"issue_ms_pipelined": [round(x, 2) for x in ts], "issue_ms_and_result_wait_ms_e2e": [[round(a, 2), round(b, 2)] for a, b in r]}))
