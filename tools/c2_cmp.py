"""C2 kernel comparison (development aid): accuracy (e1-e3 in units of u, sigma vs kernel 24) and
device time of the 16x16 FP32 register kernels on the same inputs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
from paper_2601_17979_b200.verify import verify_tensor

kernels = [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "24,34,35,36").split(",")]
u = np.finfo(np.float32).eps / 2
for fam in ("random", "arith", "geo"):
    for B in (10000, 1000, 37):
        a = gen_batch_device(fam, 16, 16, B, np.float32, kappa=1e4 if fam != "random" else 1, seed=3)
        ref = None
        for wantv in (True, False):
            opts = bs.JacobiOptions(compute_right_vectors=wantv)
            for kern in kernels:
                r = bs.solve_tensor(a, 16, 16, opts, kernel=kern); torch.cuda.synchronize()
                info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
                ts = []
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(); bs.solve_tensor(a, 16, 16, opts, kernel=kern); e1.record(); torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                line = f"{fam:6s} B={B:5d} v={int(wantv)} k={int(info['kernel'][0])} {min(ts)*1e3:7.1f} us sweeps={info['outer_sweeps'].mean():.2f} conv={info['converged'].mean():.3f}"
                if wantv:
                    e = verify_tensor(a, 16, 16, r).cpu().numpy()
                    line += f" e1={e[:,0].max()/u:.2f}u e2={e[:,1].max()/u:.2f}u e3={e[:,2].max()/u:.2f}u"
                s = r.s.double().cpu().numpy()
                if ref is None: ref = s
                line += f" |ds|/s1={np.max(np.abs(s - ref) / ref[:, :1]) / u:.2f}u"
                print(line, flush=True)
