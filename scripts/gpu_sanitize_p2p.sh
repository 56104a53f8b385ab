# compute-sanitizer over the JACC_GRAPH_P2P kernels at world 1: fused histogram/reduce/vadd+reduce ->
# allreduce, N-body -> all-gather, standalone small and large allreduce, all-gather, broadcast.
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
cat > /tmp/san_p2p.py <<'PY'
import numpy as np, sys, torch
sys.path.insert(0, ".")
import synth
import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
from paper_1508_06791_b200.torch_glue import make_graph, peer_tensor
R, W, RW = 1, 2, 3
g, _ = make_graph(0, flags=J.JACC_GRAPH_P2P | J.JACC_GRAPH_MERGE)
n = 20011
a, b = synth.vadd_inputs(n); c = np.zeros(n, np.float32); s = np.zeros(1, np.float32)
x = synth.uniform_f32(n, 4); s2 = np.zeros(1, np.float32)
keys = synth.hist_keys(n + 3); bins = np.zeros(256, np.int32)
big = synth.uniform_f32(20000, 5)
pos, vel = synth.nbody_state(700); pos2 = np.zeros_like(pos)
ALL = peer_tensor(g, (700, 4))
bc = peer_tensor(g, (333,))
g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(s, RW)])
g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s2, W)])
g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(s2, RW)])
g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(bins, W)], jacc.jacc_hist_params_t(256))
g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(bins, RW)])
g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(big, RW)])
g.add_task(J.JACC_OP_ALLGATHER, [g.a(pos, R, f32x4=True), g.a(ALL, W, f32x4=True)])
band = synth.uniform_f32(70 * 132, 6).reshape(70, 132); ext = np.zeros((74, 132), np.float32)
g.add_task(J.JACC_OP_HALO_EXCHANGE_F32, [g.a(band, R), g.a(ext, W)], jacc.jacc_halo_params_t(70, 132, 2, 0))
g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(ALL, R, f32x4=True), g.a(vel, RW, f32x4=True), g.a(pos2, W, f32x4=True)], jacc.jacc_nbody_params_t(0, 0.016, 0.01, 1.0))
g.add_task(J.JACC_OP_ALLGATHER, [g.a(pos2, R, f32x4=True), g.a(ALL, W, f32x4=True)])
g.add_task(J.JACC_OP_BROADCAST, [g.a(bc, RW)], jacc.jacc_bcast_params_t(0))
g.run(); g.run(); g.run()
print("ok", g.stats()["launches"])
g.destroy()
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_p2p.py > gpurun_out/san_p2p_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_p2p_$tool.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
