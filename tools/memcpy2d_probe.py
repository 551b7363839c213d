import time, torch
from cuda.bindings import runtime as cudart
n=16384
h=torch.empty((n,n),dtype=torch.float64,pin_memory=True)
d=torch.empty((n,n),dtype=torch.float64,device="cuda")
s=torch.cuda.Stream()
for rows in (256,1024,4096,16384):
    for kind,name in ((cudart.cudaMemcpyKind.cudaMemcpyHostToDevice,"h2d"),(cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost,"d2h")):
        torch.cuda.synchronize()
        reps=max(1,16384//rows)
        t=time.perf_counter()
        for r in range(reps):
            r0=r*rows
            if name=="h2d":
                cudart.cudaMemcpy2DAsync(d.data_ptr()+r0*8, n*8, h.data_ptr()+r0*8, n*8, rows*8, n, kind, s.cuda_stream)
            else:
                cudart.cudaMemcpy2DAsync(h.data_ptr()+r0*8, n*8, d.data_ptr()+r0*8, n*8, rows*8, n, kind, s.cuda_stream)
        torch.cuda.synchronize()
        dt=time.perf_counter()-t
        print(f"{name} segment {rows*8} B: {n*n*8/dt/1e9:.1f} GB/s", flush=True)
