"""Which part of a plane's round trip differs from the C oracle (codes / scale / zero /
fp16 output) for a given layout."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from harness import parity, synthetic  # noqa: E402
from oracle import kv_oracle as ko  # noqa: E402
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402

L, T, H, g, bits, packed = (int(a) for a in sys.argv[1:7]) if len(sys.argv) > 6 else (8, 1488, 4096, 64, 4, 1)
lay = km.KVLayout(L, T, H, 128, kind="rows", group=g, bits=bits, packed=bool(packed))
kv = synthetic.kv_job_torch(L, T, H, seed=0, job=11, group=g)
geo = lay.geometry()
print("geometry", geo)
pool = km.HostSlabPool(geo["slab_bytes"] + 4096)
eng = km.KVSwapEngine()
addr = pool.alloc(geo["slab_bytes"])
eng.offload(lay, kv, addr)
out = torch.zeros_like(kv)
eng.upload(lay, addr, out)
torch.cuda.synchronize()
slab = pool.view(addr, geo["slab_bytes"])
src = kv.cpu().numpy()
back = out.cpu().numpy()
lib = parity.c_oracle()
for p, codes, mm in parity.plane_records(lay, slab):
    if p > 2:
        break
    layer, s = divmod(p, 2)
    x = src[layer, s][None, None]
    rows = ko.view_rows(x, "contig", group=g)
    c_ref, s_ref, z_ref = parity.c_quantize(lib, rows, bits)
    c = np.asarray(codes)
    if packed:
        c = np.stack([c & 15, c >> 4], axis=1).reshape(-1)
    got = c.reshape(rows.shape)
    sc, zz = ko.params_from_minmax(mm[:, 0].astype(np.float64), -mm[:, 1].astype(np.float64), bits)
    deq = ko.dequantize_rows(c_ref, s_ref, z_ref).astype(np.float16)
    b = back[layer, s].reshape(rows.shape)
    print(p, "codes", np.array_equal(got, c_ref), int((got != c_ref).sum()), "scale", np.array_equal(sc, s_ref[:, 0]),
          "zero", np.array_equal(zz, z_ref[:, 0]), "fp16", np.array_equal(b, deq), int((b != deq).sum()),
          "first bad row", np.argwhere((got != c_ref).any(axis=1))[:3].ravel().tolist())
    bad = np.argwhere(got != c_ref)
    for r, c_ in bad[:3]:
        xr = rows[r].astype(np.float64)
        t64 = xr[c_] / s_ref[r, 0] + z_ref[r, 0]
        print("   row", r, "col", c_, "x", float(xr[c_]).hex(), "min", float(xr.min()), "max", float(xr.max()),
              "scale", float(s_ref[r, 0]).hex(), "zero", z_ref[r, 0], "x/s+z", repr(t64), "ours", int(got[r, c_]),
              "oracle", int(c_ref[r, c_]))
