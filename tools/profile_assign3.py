"""One persistent (v3) assignment at cfg5 shape for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride, stream  # noqa: E402

n, d, k = 2_000_000, 96, 64
lib = _native.lib()
_native.check(lib.csc_kmeans_tuning(b"assign_ver", 3), "tuning")
ld = row_stride(d)
f = torch.randn((n, ld), dtype=torch.float64, device="cuda")
c = torch.randn((k, ld), dtype=torch.float64, device="cuda")
fn = (f * f).sum(1)
cn = (c * c).sum(1)
lab = torch.empty(n, dtype=torch.int32, device="cuda")
own = torch.empty(n, dtype=torch.float64, device="cuda")
cnt = torch.empty(k, dtype=torch.int32, device="cuda")
for _ in range(2):
    _native.call("csc_kmeans_assign", ptr(f), ptr(fn), n, d, ld, ptr(c), ld, ptr(cn), k, ptr(lab), ptr(own),
                 ptr(cnt), stream())
torch.cuda.synchronize()
print("ok")
