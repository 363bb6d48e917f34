"""Host-side enqueue cost of one stage iteration (train_step_dev) vs its GPU time, 1 GPU.
A step is GPU-bound while the enqueue cost stays well below the GPU time; at high TP the GPU time
per step shrinks but the launch count does not."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2201_11990_b200 import planner as PL
from paper_2201_11990_b200._native import lib
from paper_2201_11990_b200.runtime import Context, Stage

tp = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = Context(0)
ctx.init_comm(bytes(128), 1, 0, 1, 1, 1, 1, 1)
if tp > 1:
    lib().mt_ctx_shard_only(ctx._h, 1)
st = Stage(ctx, PL.layer_desc(12288, 96, 2048, 1, tp_size=tp, seed=1), 1, 1)
st.init_params(1, torch.cuda.current_stream())
x = torch.randn(2048, 12288, device="cuda").bfloat16()
t = torch.randn(2048, 12288, device="cuda").bfloat16()
s = torch.cuda.current_stream()
for _ in range(3):
    st.train_step_dev(x.data_ptr(), t.data_ptr(), None, s)
torch.cuda.synchronize()
n = 20
# enqueue only (the GPU queue absorbs it as long as it does not fill up)
t0 = time.perf_counter()
for _ in range(n):
    st.train_step_dev(x.data_ptr(), t.data_ptr(), None, s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"TP shard {tp}: host enqueue {1e3 * (t1 - t0) / n:.3f} ms/step, wall {1e3 * (t2 - t0) / n:.3f} ms/step, "
      f"launches {st.launch_count()}")
