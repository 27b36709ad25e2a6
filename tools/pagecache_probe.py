"""Raw throughput of the box's 'NVMe tier' (buffered file I/O in /tmp): T
threads pread / pwrite 16 MiB pieces of a K-file striped range into one
buffer, like the engine's I/O pool; reads and writes alone and together."""
import json
import os
import sys
import tempfile
import threading
import time

import numpy as np

GB = 1 << 30
piece = 16 << 20
total = int(os.environ.get("GB", "8")) * GB
threads = int(os.environ.get("T", "16"))
files = int(os.environ.get("K", "16"))
d = tempfile.mkdtemp(dir=os.environ.get("DIR", "/tmp"))
fds = []
for k in range(files):
    p = os.path.join(d, f"f{k}")
    fd = os.open(p, os.O_RDWR | os.O_CREAT)
    os.ftruncate(fd, total // files + piece)
    os.unlink(p)
    fds.append(fd)
buf = np.ones(total, np.uint8)
mv = memoryview(buf)


def run(write, read, reps=2):
    n = total // piece
    jobs = []
    for _ in range(reps):
        for i in range(n):
            if write:
                jobs.append((True, i))
            if read:
                jobs.append((False, i))
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                if not jobs:
                    return
                w, i = jobs.pop()
            fd, off = fds[i % files], (i // files) * piece
            seg = mv[i * piece:(i + 1) * piece]
            if w:
                os.pwrite(fd, seg, off)
            else:
                os.preadv(fd, [seg], off)

    t0 = time.perf_counter()
    ts = [threading.Thread(target=worker) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    return round(reps * total * (int(write) + int(read)) / dt / 1e9, 2)


res = {"threads": threads, "files": files, "GB": total // GB}
res["write_GBps"] = run(True, False)
res["read_GBps"] = run(False, True)
res["read+write_GBps_total"] = run(True, True)
print(json.dumps(res))
