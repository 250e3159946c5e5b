"""One shape of the chained advance for an ncu capture: B rows, R steps,
random states and tokens (default: the 8-GPU share of config 5)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench_workloads as bw  # noqa: E402

from paper_2508_07014_b200 import _lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
R = int(sys.argv[2]) if len(sys.argv) > 2 else 32
tab, V = bw.table("p20k_v1024")
dt = tab.device_table(0)
rng = np.random.default_rng(5)
outs = [(torch.empty((R, B, V), dtype=torch.float32, device="cuda"),
         torch.empty((R, B, V), dtype=torch.int32, device="cuda")) for _ in range(2)]
for i in range(6):
    st = torch.from_numpy(rng.integers(0, tab.num_states, size=B).astype(np.int32)).cuda()
    tk = torch.from_numpy(rng.integers(0, V, size=(R, B)).astype(np.int32)).cuda()
    s, n = outs[i % 2]
    _lib.check(_lib.LIB.pgpb_advance_steps(dt.handle, st.data_ptr(), tk.data_ptr(), R, B, s.data_ptr(), n.data_ptr(),
                                           None, None, 0, _lib.stream_ptr()))
torch.cuda.synchronize()
print("ok")
