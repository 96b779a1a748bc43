import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2003_09446_b200 import Context
from paper_2003_09446_b200.workload import xavier_params
c = Context(0)
p = xavier_params(20, 40, seed=9)
m = c.model(20, 30, 160, 40, p)
for i in range(5):
    t = time.perf_counter(); m.update(p); dt = time.perf_counter() - t
    print("update ms", round(dt * 1e3, 2))
os.environ["DETNET_NO_JIT"] = "1"
