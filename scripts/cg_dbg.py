import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
from oracle.oracle import Port, Prob
from paper_1810_13100_b200 import datagen, ncsg
port=Port()
n=32; A=24; D=port.default_detector_count(n)
x=datagen.phantom(n,5,7); b,_=datagen.add_sinogram_noise(port.radon_forward(x,A,D),0.01,8)
rel=lambda a,b: float(np.linalg.norm(np.ravel(a)-np.ravel(b))/np.linalg.norm(np.ravel(b)))
for iters,ncg in [(1,6),(5,6),(20,6),(20,2),(20,12)]:
    prob=Prob(0,n,A,D,0.5,0.5,0.02,b)
    o=port.solve(prob,0.0,None,iters,record_every=iters,n_cg=ncg)
    p=ncsg.Problem(ncsg.CT,n,0.5,0.5,0.02,1.0,b,n_angles=A,n_det=D); p.set_cg(ncg); p.set_state()
    g=p.solve(iters,record_every=iters)
    m0=A*D
    print(iters,ncg,'x',rel(g.x[0],o.x),'us',rel(g.u[0][:m0],o.u[:m0]),'ug',rel(g.u[0][m0:],o.u[m0:]),'obj',g.rows[0][-1,1],o.rows[-1,1])
