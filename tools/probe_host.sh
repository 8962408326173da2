set -x
nproc; lscpu | head -20; free -g; nvidia-smi; 
python -c "import numpy._core._multiarray_umath as m; print([k for k,v in m.__cpu_features__.items() if v])"
python - <<'PY'
import numpy as np, math
rng=np.random.default_rng(0)
x=rng.normal(size=200000); y=rng.normal(size=200000)
a=np.arctan2(y,x); b=np.array([math.atan2(u,v) for u,v in zip(y,x)])
print("atan2 numpy vs libm mismatches", int((a!=b).sum()))
z=rng.uniform(-1,1,200000); c=np.arcsin(z); d=np.array([math.asin(t) for t in z])
print("asin mismatches", int((c!=d).sum()))
import hashlib; print("atan2 hash", hashlib.sha256(a.tobytes()).hexdigest()[:16], "asin hash", hashlib.sha256(c.tobytes()).hexdigest()[:16])
P=rng.normal(size=(100000,3)); R=np.linalg.qr(rng.normal(size=(3,3)))[0]
M=P@R.T
F=np.empty_like(M)
for j in range(3):
    pass
import numpy as np
fma=np.empty_like(M)
# emulate fma chain with math.fma
for i in range(2000):
    for j in range(3):
        fma[i,j]=math.fma(P[i,2],R[j,2],math.fma(P[i,1],R[j,1],P[i,0]*R[j,0]))
print("matmul vs fma chain mismatches (2000 rows)", int((M[:2000]!=fma[:2000]).sum()))
PY
