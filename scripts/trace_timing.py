import time, sys
sys.path.insert(0,'.')
import numpy as np
from paper_1602_05510_b200.configs import CONFIGS, make_engine
eng = make_engine(CONFIGS["C2"])
d = eng.generate_host(0, 1040)
eng.eval_trace(d[0]); eng.eval_descs(d)
for rep in range(3):
    t=time.perf_counter(); tr=eng.eval_trace(d[1]); t1=time.perf_counter()
    out,b=eng.eval_descs(d); t2=time.perf_counter()
    out,b=eng.eval_descs(d[:100]); t3=time.perf_counter()
    print(f"trace {1e3*(t1-t):.1f} ms  batch1040 {1e3*(t2-t1):.1f} ms  batch100 {1e3*(t3-t2):.1f} ms  tasks {len(tr.assignments)}")
