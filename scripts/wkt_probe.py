"""Timing breakdown of the device WKT loader on the canonical 1.31M-face ore
text: end-to-end mesh_from_wkt vs the raw host->device copy of the same
bytes (pageable and pinned) and the reference parse_wkt on the host."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_1808_09571_b200 as T  # noqa: E402

T.init(0)
ore = T.ore_body(1_000_000)
text = O.ref_serialize_mesh(ore, as_bytes=True)
n = len(text)
print(f"text {n / 1e6:.1f} MB, {len(ore)} faces")

for _ in range(2):
    T.mesh_from_wkt(text)
ts = []
for _ in range(5):
    t = time.perf_counter()
    m = T.mesh_from_wkt(text)
    ts.append(time.perf_counter() - t)
print(f"mesh_from_wkt: min {min(ts) * 1e3:.1f} ms  median {np.median(ts) * 1e3:.1f} ms")
st = T.last_stats()
print("stats", {k: v for k, v in st.items() if v})

host = torch.frombuffer(bytearray(text), dtype=torch.uint8)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pin.copy_(host)
for name, src in (("pageable", host), ("pinned", pin)):
    for _ in range(2):
        dev.copy_(src, non_blocking=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        dev.copy_(src, non_blocking=False)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"H2D {name}: {min(ts) * 1e3:.1f} ms ({n / min(ts) / 1e9:.1f} GB/s)")
t = time.perf_counter()
host2 = bytearray(text)
print(f"host memcpy: {(time.perf_counter() - t) * 1e3:.1f} ms")

m2 = T.Mesh(ore)
ts = []
for _ in range(3):
    t = time.perf_counter()
    T.Mesh(ore)
    ts.append(time.perf_counter() - t)
print(f"Mesh(upload of binary faces, {ore.nbytes / 1e6:.0f} MB): {min(ts) * 1e3:.1f} ms")

if O.REF is not None:
    t = time.perf_counter()
    O.ref_parse_wkt(text)
    print(f"reference parse_wkt (1 thread): {(time.perf_counter() - t) * 1e3:.0f} ms")

# --- H2D alternatives for the text: registering the caller's buffer, and
# multi-threaded host copies into pinned staging
import ctypes as ct  # noqa: E402
from concurrent.futures import ThreadPoolExecutor  # noqa: E402

cudart = ct.CDLL("libcudart.so.12") if False else None
buf = np.frombuffer(bytearray(text), dtype=np.uint8)
try:
    rt = torch.cuda.cudart()
    t = time.perf_counter()
    rt.cudaHostRegister(buf.ctypes.data, n, 0)
    t1 = time.perf_counter()
    reg = torch.from_numpy(buf)
    dev.copy_(reg, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(buf.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3 * (t1 - t):.1f} ms, copy {1e3 * (t2 - t1):.1f} ms, unregister {1e3 * (t3 - t2):.1f} ms")
except Exception as e:  # noqa: BLE001
    print("register failed", e)
pin_np = pin.numpy()
for nt in (1, 4, 8, 16):
    chunks = np.array_split(np.arange(n), nt)
    def cp(ix):
        pin_np[ix[0]:ix[-1] + 1] = buf[ix[0]:ix[-1] + 1]
    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(cp, chunks))
        t = time.perf_counter()
        list(ex.map(cp, chunks))
        dt = time.perf_counter() - t
    print(f"host->pinned memcpy, {nt} threads: {dt * 1e3:.1f} ms ({n / dt / 1e9:.1f} GB/s)")
import os  # noqa: E402
print("cpus", os.cpu_count())
