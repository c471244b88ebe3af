import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1908_07847_b200 as g
x, l = g.synthetic_arrays(200_000, 33, 2, "planted-linear")
net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=33, seed=3))
g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, l.astype(np.float32), 1, 0.1, g.cuda())
print("done", net.w_ih[:4])
