import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1908_07847_b200 import wide, _lib
N = int(sys.argv[1])
data = wide.WideData(N, seed=0)
torch.cuda.synchronize(); print("gen ok", N, flush=True)
w1, w2 = wide.init_wide_weights(0)
st = np.zeros((1, 3))
a, b = wide.train_wide(data, w1, w2, 1, 0.1, st)
torch.cuda.synchronize(); print("train ok", N, st, flush=True)
