"""Per-CTA timeline of the fused decode at C3 (diagnostics): needs a library built with
-DQJL_UD_TRACE=1 (tools/build_variant.sh trace "-DQJL_UD_TRACE=1"; QJL_LIB=variants/libqjl_trace.so).
Prints, per launch wave (CTA index // SMs), when CTAs leave griddepcontrol.wait, finish
their main loop and exit, relative to the first CTA's wait -- for the PDL-chained step
(prep + decode, as timed by bench.py) and for the decode launched alone."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2406_03482_b200 import _lib

w = dict(bench.WORKLOADS["c3"])
dev = torch.device("cuda", 0)
from paper_2406_03482_b200.distributed import shard_units
sh = shard_units(64, 1, 0)
cache = bench.build_cache(w, sh, 0, dev)
q = bench.make_queries(w, sh, 0, dev)
U, d, G = w["batch"] * w["kv_heads"], w["d"], w["G"]
out = torch.empty(U, G, d, device=dev)
lib = _lib.load()
fn = lib.qjl_debug_ud_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
sms = torch.cuda.get_device_properties(0).multi_processor_count
C = 4 * sms
res = {}
for mode in ("chained_step", "kernel_chain", "deterministic"):
    for i in range(20):
        if mode == "chained_step":
            cache.decode(q, out=out, chained=i > 0)
        elif mode == "kernel_chain":
            cache.bench_decode_kernel(q, reps=3, out=out)
        else:
            cache.decode(q, out=out, deterministic=True)
    torch.cuda.synchronize()
    buf = np.zeros((C, 4), np.uint64)
    assert fn(buf.ctypes.data, C) == 0
    t = buf[:, :3].astype(np.float64)
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3
    r = {}
    for wv in range(4):
        sl = t[wv * sms:(wv + 1) * sms]
        r[f"wave{wv}"] = {"wait": [round(float(sl[:, 0].min()), 2), round(float(sl[:, 0].max()), 2)],
                          "loop_done": [round(float(sl[:, 1].min()), 2), round(float(np.median(sl[:, 1])), 2), round(float(sl[:, 1].max()), 2)],
                          "end": [round(float(sl[:, 2].min()), 2), round(float(np.median(sl[:, 2])), 2), round(float(sl[:, 2].max()), 2)]}
    r["kernel_end"] = round(float(t[:, 2].max()), 2)
    sm = buf[:, 3].astype(np.int64)
    per_sm_loop = np.array([t[sm == i, 1].max() for i in np.unique(sm)])
    per_sm_first = np.array([t[sm == i, 1].min() for i in np.unique(sm)])
    per_sm_mean = np.array([t[sm == i, 1].mean() for i in np.unique(sm)])
    r["same_sm_as_c_plus_148j"] = [round(float(np.mean(sm[:C - 148 * j] == sm[148 * j:])), 3) for j in (1, 2, 3)]
    r["smid_first8"] = sm[:8].tolist()
    r["ctas_per_sm"] = sorted(set(np.bincount(sm).tolist()) - {0})
    r["sm_last_loop_done_pct"] = [round(float(x), 2) for x in np.percentile(per_sm_loop, [0, 10, 50, 90, 100])]
    r["sm_first_loop_done_pct"] = [round(float(x), 2) for x in np.percentile(per_sm_first, [0, 10, 50, 90, 100])]
    r["sm_mean_loop_done_pct"] = [round(float(x), 2) for x in np.percentile(per_sm_mean, [0, 10, 50, 90, 100])]
    r["loop_done_pct"] = [round(float(x), 2) for x in np.percentile(t[:, 1], [0, 10, 50, 90, 100])]
    r["end_pct"] = [round(float(x), 2) for x in np.percentile(t[:, 2], [0, 10, 50, 90, 99, 100])]
    r["mean_loop_done"] = round(float(t[:, 1].mean()), 2)
    if hasattr(lib, "qjl_debug_ud_stat"):
        st = np.zeros((C, 4), np.uint64)
        lib.qjl_debug_ud_stat.argtypes = [ctypes.c_void_p, ctypes.c_int]
        assert lib.qjl_debug_ud_stat(st.ctypes.data, C) == 0
        st = st.astype(np.float64)
        ghz = 1.9
        r["tiles_pct"] = [float(x) for x in np.percentile(st[:, 0], [0, 50, 100])]
        r["runs_mean"] = round(float(st[:, 3].mean()), 2)
        r["issue_us_per_tile"] = round(float((st[:, 1] / np.maximum(st[:, 0], 1)).mean() / ghz / 1e3), 3)
        r["fullwait_us_per_tile"] = round(float((st[:, 2] / np.maximum(st[:, 0], 1)).mean() / ghz / 1e3), 3)
        r["loop_us_per_tile"] = round(float((t[:, 1] - t[:, 0]).sum() / st[:, 0].sum()), 3)
    res[mode] = r
for k, r in res.items():
    print(k, {kk: v for kk, v in r.items() if not kk.startswith("wave")})
    for wv in range(4):
        print("  ", wv, r[f"wave{wv}"])
