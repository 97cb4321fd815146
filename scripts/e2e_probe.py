"""Device-resident vs host-buffer (e2e) evaluation of one preset, with the
engine's own kernel timings (dev tool).  usage: e2e_probe.py <preset> <batch>"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1602_05510_b200.configs import CONFIGS, make_engine  # noqa: E402
from paper_1602_05510_b200.engine import DESC_DTYPE, OUTCOME_DTYPE  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
eng = make_engine(CONFIGS[name])
print("chunk", eng.info().chunk if hasattr(eng.info(), "chunk") else "?")
descs = torch.empty(B * DESC_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
outs = torch.empty(B * OUTCOME_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
host = eng.generate_host(0, B)
eng.generate_device(0, B, descs.data_ptr(), st.cuda_stream)
st.synchronize()
for rep in range(3):
    t = time.perf_counter()
    b = eng.eval_descs_device(descs.data_ptr(), B, 0, outs.data_ptr(), st.cuda_stream)
    st.synchronize()
    dt = time.perf_counter() - t
    print(f"device: {1e3*dt:.1f} ms wall, kernels {b.kernel_ms:.1f} (build {b.build_ms:.1f}, sim {b.sim_ms:.1f})")
    t = time.perf_counter()
    out, b2 = eng.eval_descs(host, first=0)
    dt = time.perf_counter() - t
    print(f"host:   {1e3*dt:.1f} ms wall, kernels {b2.kernel_ms:.1f} (build {b2.build_ms:.1f}, sim {b2.sim_ms:.1f})")
