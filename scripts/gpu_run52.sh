python -c "import __graft_entry__ as g; g.build()" > /dev/null
cat > /tmp/cv.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, synth
import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
from paper_1508_06791_b200.torch_glue import make_graph
img = synth.uniform_f32(256*256, 1, -1, 1).reshape(256, 256); f = synth.uniform_f32(25, 2).reshape(5, 5); out = np.zeros_like(img)
g, _ = make_graph(0)
g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img, 1), g.a(f, 1), g.a(out, 2)], jacc.jacc_conv2d_params_t(256, 256, 2, 0))
g.run(); print("ok")
PY
timeout 300 compute-sanitizer --tool memcheck --show-backtrace no python /tmp/cv.py 2>&1 | head -12
cuobjdump -sass build/jacc/conv2d.cu.o | awk '/Function :/{p=($0 ~ /conv2d_tma_kernelILi2E/)} p' | head -120 > gpurun_out/cv2.sass
