"""cfg2: how much of the degree walk's stationary visits the hottest bucket lines hold (pi(v) ~ deg(v) T(v)).
Measured (CPU): 100 MB of buckets hold 10 % of the visits, 1 GB 41 %, so an L2-resident hot set cannot
carry the walk -- each step stays a DRAM round trip."""
import numpy as np, sys
sys.path.insert(0, '/root/repo')
from synth import rmat_csr
g = rmat_csr(4_800_000, 69_000_000, 2)
rp = g.row_ptr.numpy(); col = g.col_idx.numpy().view(np.uint32)
deg = np.diff(rp).astype(np.float64)
T = np.add.reduceat(deg[col], rp[:-1][deg > 0])
Tv = np.zeros(len(deg)); Tv[deg > 0] = T
pi = deg * Tv; pi /= pi.sum()
nb = np.where(deg > 0, np.floor(np.log2(np.maximum(Tv / np.maximum(deg, 1), 1))), 0)
W = 2.0 ** nb
nbk = np.where(deg > 0, np.floor((Tv - 1) / W) + 1, 0)
bytes_v = nbk * 128
order = np.argsort(-pi / np.maximum(bytes_v, 1))   # hottest per byte first
cp = np.cumsum(pi[order]); cb = np.cumsum(bytes_v[order])
for mb in (32, 64, 100, 200, 500, 1000, 4000):
    i = np.searchsorted(cb, mb * 1e6)
    print(f"{mb:5d} MB of buckets hold {cp[min(i, len(cp)-1)]*100:.1f} % of the walk's visits")
print("total bucket GB", cb[-1] / 1e9, "max deg", deg.max())
