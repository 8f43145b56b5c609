"""Per-CTA timeline of the 2048-bit headline kernel (diagnostic; tools/cta_times.cu): for batches
of 1, 2 and 4.61 waves, the CTA durations by wave (launch order) and by SM.  One JSON line each."""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2410_18129_b200 import inputs as I  # noqa: E402
from paper_2410_18129_b200 import mpb  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libcta_times.so"))
lib.cta_modexp_2048.restype = ctypes.c_int
lib.cta_modexp_2048.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
for count in [int(x) for x in (sys.argv[1:] or ["56832", "113664", "262144"])]:
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=2048)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, R2 = mpb.mont_batch_setup(dN, 2048)
    ws = mpb.modexp_workspace(count, 2048, 5, 0)
    out = mpb.empty_sliced(64, count)
    torch.cuda.synchronize()
    args = [x.data_ptr() for x in (dN, Np, R2, dB, dE, out)] + [count, 5, ws.data_ptr()]
    for rep in range(2):
        rc = lib.cta_modexp_2048(*args)
        assert rc == 0, rc
    g = (count + 127) // 128
    t0 = (ctypes.c_ulonglong * g)(); t1 = (ctypes.c_ulonglong * g)(); sm = (ctypes.c_uint32 * g)()
    lib.cta_times_take(t0, t1, sm, g)
    t0 = np.array(t0, np.float64); t1 = np.array(t1, np.float64); sm = np.array(sm)
    base_t = t0.min()
    s, e = (t0 - base_t) / 1e6, (t1 - base_t) / 1e6
    d = e - s
    order = np.argsort(s, kind="stable")
    waves = []
    slots = 444
    for wv in range(0, g, slots):
        idx = order[wv:wv + slots]
        waves.append({"wave": wv // slots, "ctas": int(len(idx)), "start_ms": [round(float(s[idx].min()), 2), round(float(s[idx].max()), 2)],
                      "dur_ms": [round(float(d[idx].min()), 2), round(float(np.median(d[idx])), 2), round(float(d[idx].max()), 2)]})
    per_sm = np.zeros(int(sm.max()) + 1)
    for i in range(g):
        per_sm[sm[i]] = max(per_sm[sm[i]], e[i])
    print(json.dumps({"count": count, "ctas": g, "launch_ms": round(float(e.max()), 2), "waves": waves,
                      "sm_end_ms": [round(float(per_sm.min()), 2), round(float(np.median(per_sm)), 2), round(float(per_sm.max()), 2)]}))
    sys.stdout.flush()
