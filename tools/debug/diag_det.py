import sys, hashlib, numpy as np
sys.path.insert(0,'.')
import paper_2408_02937_b200 as bivf
x = bivf.synthetic_dataset(1_010_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
print('data sha', hashlib.sha1(x.tobytes()).hexdigest()[:12])
base = x[:1_000_000]
c1,a1,i1 = bivf.kmeans(base[:100000], 1024, 10, 42)
print('cent sha', hashlib.sha1(c1.tobytes()).hexdigest()[:12], 'asg sha', hashlib.sha1(a1.tobytes()).hexdigest()[:12], i1)
c3,a3,i3 = bivf.kmeans(base[:100000], 1024, 0, 42)
print('seed-only sha', hashlib.sha1(c3.tobytes()).hexdigest()[:12])
