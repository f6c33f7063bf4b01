import sys, numpy as np, hashlib, platform
sys.path.insert(0,'oracle'); import oracle as O
c1=np.load('gpurun_out/c1.npy'); q=np.load('gpurun_out/q.npy')
orc = O.OracleIndex(c1, c1[:1], np.zeros(1, np.uint32), 1024, 16)
P=np.array([orc.probes(q[j],32) for j in range(50)])
print(platform.processor(), hashlib.sha1(P.tobytes()).hexdigest()[:12])
print(hashlib.sha1(open('oracle/liboracle.so','rb').read()).hexdigest()[:12])
k=np.array([O.oracle_l2(q[0], c) for c in c1[:8]], np.float32); print(k)
