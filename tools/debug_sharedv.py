"""Debug: shared-V vs private-V request on the tiny model (which rows differ)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2601_12904_b200 import fusion as F

ratio = float(sys.argv[1]) if len(sys.argv) > 1 else 0.15
eng = F.Engine("tiny", seed=4321)
c = eng.cfg
print("cfg", c.layers, c.d_model, c.n_heads, c.n_kv_heads, c.head_dim)
store = F.ChunkKVStore(c)
rng = np.random.default_rng(5)
system = rng.integers(0, c.vocab, 8).tolist()
lens = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256, 200, 333, 97, 256, 150]
chunks = [rng.integers(0, c.vocab, n).tolist() for n in lens]
ids = [eng.preprocess_isolated(store, ch, system=system) for ch in chunks]
q = rng.integers(0, c.vocab, 32).tolist()
T = len(system) + sum(lens) + 32
out = []
for sh in (True, False):
    F.set_shared_v(sh)
    res = F.Result(eng, T + 16)
    eng.reprocess(store, q, ids, ratio, res, system=system)
    k, v = res.fused_kv()
    out.append((res.logits().copy(), res.crit().copy(), k, v, res.memory()))
(la, ca, ka, va, ma), (lb, cb, kb, vb, mb) = out
print("mem", ma, mb, "crit equal", np.array_equal(ca, cb), "k", len(ca))
print("logits rel", float(np.linalg.norm(la - lb) / np.linalg.norm(lb)))
for l in range(c.layers):
    dk = np.nonzero((ka[l] != kb[l]).any(axis=(1, 2)))[0]
    dv = np.nonzero((va[l, :T] != vb[l, :T]).any(axis=(1, 2)))[0]
    crit0 = set((ca - 1).tolist())
    print(f"layer {l}: K rows differ {len(dk)} (first {dk[:10].tolist()}), V rows differ {len(dv)} "
          f"(first {dv[:10].tolist()}, in crit {sum(int(x) in crit0 for x in dv)}, >=T-32 {int((dv >= T - 32).sum())})")
