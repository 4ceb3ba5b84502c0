import numpy as np, sys
sys.path.insert(0, '.')
import paper_2604_00546_b200 as hd, oracle
for log_n in (12, 15, 16):
    ctx = hd.Context(log_n, 3); o = oracle.Oracle(log_n, 3)
    rng = np.random.default_rng(log_n)
    for l, m in enumerate(o.p.moduli):
        row = rng.integers(0, m, o.n, dtype=np.uint64)[None]
        f = ctx.test_ntt(row, [l])[0]; i = ctx.test_ntt(row, [l], inverse=True)[0]
        fo = o.ntt(row[0], l); io = o.ntt(row[0], l, inverse=True)
        print(log_n, l, m.bit_length(), "fwd", (f == fo).mean(), "inv", (i == io).mean(), "inv-fwd roundtrip", (ctx.test_ntt(i[None], [l])[0] == row[0]).mean(), flush=True)
        if not (i == io).all():
            bad = np.nonzero(i != io)[0][:5]; print("   bad idx", bad, i[bad], io[bad], flush=True)
