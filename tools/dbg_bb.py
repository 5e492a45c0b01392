import numpy as np, sys
sys.path.insert(0, "/root/repo")
import paper_1708_08427_b200 as rq
for d in ([0,0,1.0],[0,0,-1.0],[0.3,0.2,0.9],[1.0,0,0]):
    f = rq.factor_bead_bead(d)
    print(d, f.t22.ravel(), f.omega.ravel()[:3])
m = np.array([[np.sqrt(2),0,0],[0,np.sqrt(2),0],[0,0,0.0]])
print(rq.small_lq(m)[0].ravel())
