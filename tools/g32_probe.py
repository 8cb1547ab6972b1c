"""INT4 / INT8 g32 quantize on each codec kernel family (FC_CODEC_QKERNEL=lane|gq|gpl|auto in the
environment), CUDA-graph device time over bf16 [8,1024,8192], bit-exact against the default."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from bench import graph_time  # noqa: E402

M = 8 * 1024 * 8192
torch.manual_seed(0)
x = torch.randn(M, device="cuda").to(torch.bfloat16)
st = torch.cuda.current_stream()
for bits in (4, 8):
    cc = fc.CodecConfig(bits=bits, group_size=32)
    L = cc.device_layout(M)
    buf = torch.empty(L.total_bytes, dtype=torch.uint8, device="cuda")
    c = cc.to_fc()
    qf = lambda: _lib.check(_lib.lib().fc_quantize(x.data_ptr(), _lib.DTYPE_BF16, M, C.byref(c), buf.data_ptr(),  # noqa: E731
                                                   None, torch.cuda.current_stream().cuda_stream))
    qf()
    torch.cuda.synchronize()
    ref = torch.load("/tmp/g32_%d.pt" % bits) if os.path.exists("/tmp/g32_%d.pt" % bits) else None
    if ref is None:
        torch.save(buf.cpu(), "/tmp/g32_%d.pt" % bits)
    ok = ref is None or torch.equal(ref, buf.cpu())
    t = graph_time(qf, 10, st)
    alg = 2 * M + L.wire_bytes
    print(f"{os.environ.get('FC_CODEC_QKERNEL', 'auto')} int{bits} g32: {t*1e3:.1f} us  "
          f"{alg / (t * 1e-3) / 1e9 / 6551:.3f} of HBM  bitexact {ok}", flush=True)
