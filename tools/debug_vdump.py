"""Debug: compare the patched V tiles the attention kernel consumed
(FRAG_VPATCH_DUMP) with the private fused V (tiny model, r given)."""
import os
import sys
import numpy as np
sys.path.insert(0, ".")
ratio = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
dump = "/tmp/vdump.bin"
if os.path.exists(dump):
    os.remove(dump)
os.environ["FRAG_VPATCH_DUMP"] = dump
from paper_2601_12904_b200 import fusion as F

eng = F.Engine("tiny", seed=4321)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(5)
system = rng.integers(0, c.vocab, 8).tolist()
lens = [256, 200, 333, 97, 256, 150]
chunks = [rng.integers(0, c.vocab, n).tolist() for n in lens]
ids = [eng.preprocess_isolated(store, ch, system=system) for ch in chunks]
q = rng.integers(0, c.vocab, 32).tolist()
T = len(system) + sum(lens) + 32
F.set_shared_v(False)
res = F.Result(eng, T + 16)
eng.reprocess(store, q, ids, ratio, res, system=system)
kp, vp = res.fused_kv()
F.set_shared_v(True)
res2 = F.Result(eng, T + 16)
eng.reprocess(store, q, ids, ratio, res2, system=system)
crit = set((res2.crit() - 1).tolist())
raw = open(dump, "rb").read()
off = 0
launch = 0
while off < len(raw):
    hdr = np.frombuffer(raw[off:off + 32], dtype=np.int32)
    off += 32
    M, ns, Hkv, dh, G, layer, sk, dual = [int(x) for x in hdr]
    nqb = (M + 128 // G - 1) // (128 // G)
    nbytes = ns * nqb * Hkv * 8 * 128 * dh * 2
    data = np.frombuffer(raw[off:off + nbytes], dtype=np.uint16).reshape(ns, nqb * Hkv, 8, 128, dh)
    off += nbytes
    bad = 0
    tot = 0
    for z in range(ns):
        for x in range(nqb * Hkv):
            hk = x % Hkv
            for j in range(8):
                key0 = (z * sk if ns > 1 else 0) + j * 128
                tile = data[z, x, j]
                if not tile.any():
                    continue
                # unswizzle: row r, 16B chunk cc at r*128 + ((cc ^ (r&7))<<4) within each 64-col atom
                un = np.zeros_like(tile)
                t8 = tile.reshape(128, dh // 8, 8)
                for r in range(128):
                    for cc in range(dh // 8):
                        at, c8 = cc // 8, cc % 8
                        src = (at * 128 * 64 + r * 64 + ((c8 ^ (r & 7)) * 8))
                        un[r, cc * 8:(cc + 1) * 8] = tile.reshape(-1)[src:src + 8]
                for r in range(128):
                    row = key0 + r
                    if row >= T or row in crit:
                        continue
                    tot += 1
                    if not np.array_equal(un[r], vp[layer, row, hk]):
                        bad += 1
                        if bad <= 5:
                            print(f"  launch {launch} L{layer} z{z} x{x} j{j} row {row} differs")
    print(f"launch {launch}: M={M} splits={ns} dual={dual} layer={layer}: {bad} of {tot} rows differ")
    launch += 1
    if launch >= 4:
        break
