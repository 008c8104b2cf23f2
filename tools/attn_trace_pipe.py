"""Per-tile timeline of the sparse-pass attention inside a real request
(FRAG_ATTN_TRACE, eager launches): CTA 0 of each Q-in-TMEM launch -- S ready,
P done, S / PV issue (MMA warp) and, with shared V pages, the patch warp's
'primary box landed' stamp and patch-row count. Usage: [config] [ratio]."""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "attn_trace.bin")
os.environ["FRAG_ATTN_TRACE"] = path
os.environ["FRAG_GRAPHS"] = "0"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2601_12904_b200 import fusion as F  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
ratio = float(sys.argv[2]) if len(sys.argv) > 2 else 0.15
shared = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
F.set_shared_v(shared)
eng = F.Engine(cfg, seed=1)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, c.vocab, 2048).tolist()) for _ in range(8)]
q = rng.integers(0, c.vocab, 32).tolist()
res = F.Result(eng, 8 * 2048 + 32)
eng.reprocess(store, q, ids, ratio, res)
res.sync()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4, 256, 4).astype(np.int64)
print(f"{len(rec)} traced launches; shared V {shared}")
med = lambda x: float(np.median(x)) if len(x) else float("nan")  # noqa: E731
for li, r in enumerate(rec):
    a, b, c2, c3 = r[0], r[1], r[2], r[3]
    n = int((a[:, 0] > 0).sum())
    if n < 40:
        continue
    s_ready, p_done, s_iss, pv_iss = (a[:n, i] for i in range(4))
    raw = b[:n, 3]
    land = raw & 0xffffffffffff
    rows = raw >> 48
    print(f"launch {li}: tiles {n}; period {med(np.diff(s_ready)):.0f} cyc; P done -> PV issue "
          f"{med(pv_iss - p_done):.0f}; S issue -> S ready {med(s_ready - s_iss):.0f}")
    v_iss, v_land, stg_land, v_rdy = c2[:n, 0], c2[:n, 1] & 0xffffffffffff, c2[:n, 2], c2[:n, 3]
    run = c2[:n, 1] >> 48
    if v_iss.any():
        t0 = s_ready[0]
        for u in range(min(n, 12)):
            print(f"   tile {u:3d}: V issue {v_iss[u]-t0:7d} landed {v_land[u]-t0:7d} staged {stg_land[u]-t0 if stg_land[u] else -1:7d}"
                  f" ready {v_rdy[u]-t0:7d} | S ready {s_ready[u]-t0:7d} P done {p_done[u]-t0:7d} PV issue {pv_iss[u]-t0:7d} run {run[u]}")
        scat, top = c3[:n, 0], c3[:n, 1]
        print(f"   medians: staged->scattered {med(scat - stg_land):.0f}, scattered->ready(fence) {med(v_rdy - scat):.0f}, "
              f"prev ready->loop top done {med(top[1:] - v_rdy[:-1]):.0f}, top->landed {med(v_land - top):.0f}")
        print(f"   medians: V issue->landed {med(v_land - v_iss):.0f}, landed->ready {med(v_rdy - v_land):.0f}, "
              f"ready->PV issue {med(pv_iss - v_rdy):.0f}, P done->PV {med(pv_iss - p_done):.0f}")
    if land.any():
        print(f"   V primary landed -> PV issue {med(pv_iss - land):.0f} cyc (p10 {np.percentile(pv_iss - land, 10):.0f},"
              f" p90 {np.percentile(pv_iss - land, 90):.0f}); PV issue - P done > 0 on {int((pv_iss > p_done + 50).sum())}"
              f" tiles; patch rows median {med(rows):.0f} max {int(rows.max())}")
        print(f"   land - P done: median {med(land - p_done):.0f} (negative = V ready before P)")
    if li > 40:
        break
