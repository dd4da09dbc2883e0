OUT=gpurun_out/g19; mkdir -p $OUT
N="--kernel-name-base demangled"
ncu --profile-from-start off --set full --clock-control none --import-source on $N -k 'regex:k_gemm' -o $OUT/call_gemms python tools/profile_call.py 2 > $OUT/ncu_call.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv python tools/profile_call.py 2 > $OUT/ncu_launch.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg4.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np, paper_2211_00696_b200 as pq
from paper_2211_00696_b200.workloads import config, allen_cahn_u0
w=config(4); a=pq.KroneckerSum(w.A); u0=torch.from_numpy(allen_cahn_u0(w.N)).cuda()
for i in range(3): pq.integrate(a, ('cubic',1.0,-1.0), u0, 0.0, 5*w.tau, 5, pq.etdrk4_tableau(), pq.PhiRequest(eps=w.eps))
torch.cuda.synchronize(); torch.cuda.cudart().cudaProfilerStart()
pq.integrate(a, ('cubic',1.0,-1.0), u0, 0.0, 5*w.tau, 5, pq.etdrk4_tableau(), pq.PhiRequest(eps=w.eps)); torch.cuda.synchronize(); torch.cuda.cudart().cudaProfilerStop()
" > $OUT/ncu_launch4.log 2>&1
ls -la $OUT
