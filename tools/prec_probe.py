import ctypes, os, sys, numpy as np, torch
R=os.environ.get("GRAFT_REPO_ROOT","/root/repo"); sys.path.insert(0,R); sys.path.insert(0,R+"/tests")
lib=ctypes.CDLL(R+"/tests/cuda/libumma_probe.so")
lib.umma_probe.restype=ctypes.c_int
lib.umma_probe.argtypes=[ctypes.c_void_p]*3+[ctypes.c_int]*2
K,N=2048,128
g=torch.Generator(device="cuda").manual_seed(5)
for trial in range(3):
    A=(torch.rand(128,K,device="cuda",generator=g)*2-1).half()
    B=torch.randn(N,K,device="cuda",generator=g).half()
    D=torch.zeros(128,N,device="cuda")
    assert lib.umma_probe(A.data_ptr(),B.data_ptr(),D.data_ptr(),K,N)==0
    ex=(A.double()@B.double().T)
    e_tc=(D.double()-ex).abs()
    # fp32 sequential accumulation on CPU
    a=A.float().cpu().numpy(); b=B.float().cpu().numpy()
    acc=np.zeros((128,N),np.float32)
    for k in range(K): acc+= np.outer(a[:,k],b[:,k]).astype(np.float32)
    e_32=np.abs(acc.astype(np.float64)-ex.cpu().numpy())
    print("trial",trial,"tc max %.2e mean %.2e | fp32-seq max %.2e mean %.2e | |D| mean %.1f"%(e_tc.max(),e_tc.mean(),e_32.max(),e_32.mean(),ex.abs().mean()))
import paper_1907_05124_b200 as mb
from conftest import golden
gd=golden("sweeps")
for name,n,J in [("sk2000",2000,mb.gen_sk_gaussian(2000,7)),("pm256",256,mb.gen_sk_pm1(256,1))]:
    for kern,small in [("dense_umma","0"),("dense_simt",None)]:
        if small: os.environ["MARS_DENSE_SMALL"]=small
        else: os.environ.pop("MARS_DENSE_SMALL",None)
        p=mb.IsingProblem.dense(n,J,kernel=kern)
        s0=np.stack([mb.initial_state(int(s),n) for s in gd[name+"_seeds"]]).astype(np.float32)
        for ti,T in enumerate(gd[name+"_temps"]):
            out,k=mb.debug_sweep(p,s0,float(T),1)
            err=np.abs(out.astype(np.float64)-gd[name+"_out"][ti]).max(axis=1)
            print(name,kern,T,"max|ds| per state", " ".join("%.1e"%e for e in err))
