"""Small SGEMM shapes through the C-ABI with a NaN-filled device C:
prints whether C was written and the max error vs numpy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
from paper_1508_06791_b200.torch_glue import make_graph
import synth
for (M, N, K, dist) in [(128, 256, 16, "int"), (128, 256, 16, "eye"), (128, 256, 256, "int"), (256, 256, 256, "int"),
                        (128, 256, 32, "int")]:
    if dist == "eye":
        A = np.zeros((M, K), np.float32); A[np.arange(K), np.arange(K)] = 1
        B = np.arange(K * N, dtype=np.float32).reshape(K, N) % 7
    else:
        A, B = synth.sgemm_inputs(M, N, K, "int", seed=5)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.full((M, N), float("nan"), device="cuda")
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_SGEMM_F32, [g.a(dA, 1), g.a(dB, 1), g.a(dC, 2)],
               jacc.jacc_sgemm_params_t(M, N, K, K, N, N, J.JACC_SGEMM_3XTF32, 0))
    g.run(); g.destroy()
    C = dC.cpu().numpy()
    R = A.astype(np.float64) @ B.astype(np.float64)
    print(M, N, K, dist, "nan:", int(np.isnan(C).sum()), "zeros:", int((C == 0).sum()), "of", C.size,
          "maxerr:", float(np.nanmax(np.abs(C - R))), "C[0,:8]", C[0, :8], "R[0,:8]", R[0, :8], flush=True)
    if dist == "eye":
        # which B element landed where: C[i, j] should be B[i, j]
        for i in range(3):
            print("  row", i, "C", C[i, :40:4], "B", B[i, :40:4])
