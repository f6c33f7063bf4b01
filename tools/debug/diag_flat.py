import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import paper_2408_02937_b200 as bivf
import oracle as O
for C in (32, 64, 96, 128, 160, 256, 1024):
  for D in (8, 128):
    cent = bivf.synthetic_dataset(C, D, C, 5)
    q = bivf.synthetic_dataset(200, D, C, 6)
    ix = bivf.ClusterIndex.empty(D, C, block_capacity=64, num_blocks=16)
    ix.set_centroids(cent)
    orc = O.OracleIndex(cent, cent[:1], np.zeros(1, np.uint32), 64, 16)
    for P in (1, 8, 32):
      for nq in (1, 37, 200):
        pr = ix.probes(q[:nq], P)
        bad = sum(int(not np.array_equal(orc.probes(q[j], P), pr[j])) for j in range(nq))
        if bad: print('C', C, 'D', D, 'P', P, 'nq', nq, 'bad', bad, pr[0][:4], orc.probes(q[0], P)[:4])
print('done')
