"""One merge launch of a given shape (for `ncu --set full`): python tools/merge_one.py ROWS COLS RANK [BATCH]
(BATCH > 1: one pb_op_merge_batch launch over BATCH tensors of that shape). Weights random bf16 on the device."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_17707_b200 import _binding as B  # noqa: E402

rows, cols, rank = (int(x) for x in sys.argv[1:4])
nb = int(sys.argv[4]) if len(sys.argv) > 4 else 1
Ws = [(torch.randn(rows, cols, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(nb)]
Bf = (torch.randn(rows, rank, device="cuda") * 0.01).to(torch.bfloat16)
Af = (torch.randn(rank, cols, device="cuda") * 0.01).to(torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    if nb == 1:
        B.pb_op_merge(Ws[0].data_ptr(), cols, rows, cols, Bf.data_ptr(), Af.data_ptr(), rank, 2.0, s)
    else:
        B.pb_op_merge_batch([w.data_ptr() for w in Ws], [cols] * nb, [rows] * nb, [cols] * nb, [Bf.data_ptr()] * nb,
                            [Af.data_ptr()] * nb, rank, [2.0] * nb, s)
torch.cuda.synchronize()
print("ok", rows, cols, rank, nb)
