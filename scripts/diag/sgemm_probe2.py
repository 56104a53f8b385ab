import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
from paper_1508_06791_b200.torch_glue import make_graph
M, N, K = 128, 256, 16
A = np.zeros((M, K), np.float32); A[np.arange(K), np.arange(K)] = 1
A[0, :] = np.arange(K) + 0.5
B = (np.arange(K * N, dtype=np.float32).reshape(K, N) % 97) + 0.25
dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
dC = torch.full((M, N), float("nan"), device="cuda")
g, _ = make_graph(0)
g.add_task(J.JACC_OP_SGEMM_F32, [g.a(dA, 1), g.a(dB, 1), g.a(dC, 2)],
           jacc.jacc_sgemm_params_t(M, N, K, K, N, N, J.JACC_SGEMM_3XTF32, 0))
g.run(); g.destroy()
C = dC.cpu().numpy()
print("C[0,:8]", C[0, :8], "ref", (A.astype(np.float64) @ B)[0, :8])
print("C[1,:8]", C[1, :8], "ref", B[1, :8])
