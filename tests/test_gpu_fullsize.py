"""Full-size parity at the BASELINE configs against the UNMODIFIED reference.

`tests/golden/digests.json` holds sha256 digests that
`tests/golden/make_golden.py digests` computed from the reference itself
(`qcollectives.flash_all_reduce`, collectives.py:321-402) on
`gen_rank_activations(ActivationProfile(hidden, tokens, seed=0), N)`
(workload.py:111-120) rounded to the config's dtype:

* every rank's input (proves the GPU box regenerates the same inputs),
* the float32 output (all ranks are identical in the reference),
* for every directed pair s -> j, the stage-1 wire messages the reference
  sent (codes | fp16 scales | zero points, each concatenated over pieces),
* for every owner j, its stage-2 payload.

Here the same inputs go through the CUDA path (all ranks as logical ranks of
cuda:0) and EVERY output, EVERY stage-1 receive slot and EVERY stage-2 gather
slot is compared bit for bit (digest equality). bf16/fp16 outputs must equal
the round-to-nearest-even of the float32 output (0 ulp).
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle import flash_oracle as orc

pytestmark = pytest.mark.gpu

fc = pytest.importorskip("paper_2412_04964_b200")
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

DIGESTS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "digests.json")


def _digests():
    with open(DIGESTS) as fh:
        return json.load(fh)


def sha(t) -> str:
    if isinstance(t, torch.Tensor):
        t = t.detach().contiguous().cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(t).view(np.uint8).tobytes()).hexdigest()


def inputs_for(d):
    xs = orc.gen_rank_activations(d["hidden"], d["tokens"], d["seed"], d["n"])
    rnd = orc.round_to_bf16 if d["dtype"] == "bf16" else orc.round_to_fp16
    xs = [rnd(x).ravel() for x in xs]
    for r, x in enumerate(xs):
        assert sha(x.astype(np.float32)) == d["inputs"][r], f"input of rank {r} differs from the reference's"
    return xs


MODES = {"split": 0, "fused": 1}


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("name", ["c1_tp4_int8_fp16", "tp8_int8_bf16", "tp8_int6_bf16", "c2_tp8_int4_bf16"])
def test_fullsize_vs_reference_digests(name, mode):
    d = _digests()[name]
    n, m = d["n"], d["m"]
    xs = inputs_for(d)
    tdt = torch.bfloat16 if d["dtype"] == "bf16" else torch.float16
    ts = [torch.from_numpy(x).cuda().to(tdt) for x in xs]
    del xs
    cfg = fc.FlashConfig.from_bits(d["bits"])
    seg = m // n
    comm = FlashComm.local([0] * n, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    try:
        comm.set_option(_lib.OPT_FUSED, MODES[mode])
        outs = comm.all_reduce_local(ts, cfg, out_dtype=torch.float32)
        for r in range(n):
            assert sha(outs[r]) == d["out_f32"], f"float32 output of rank {r}"
        # every stage-1 receive slot s -> j and every stage-2 gather slot (owner j at rank p)
        for j in range(n):
            for s in range(n):
                if s == j:
                    continue
                q = comm.slot(j, 1, s, cfg.stage1_codec)
                got = [sha(q.codes), sha(q.scales_f16.view(torch.uint8)), sha(q.zeros)]
                assert got == d["stage1"][f"{s}->{j}"], f"stage-1 slot {s}->{j}"
                q2 = comm.slot(s, 2, j, cfg.stage2_codec)
                got2 = [sha(q2.codes), sha(q2.scales_f16.view(torch.uint8)), sha(q2.zeros)]
                assert got2 == d["stage2"][str(j)], f"stage-2 payload of owner {j} at rank {s}"
        ref32 = outs[0].clone()
        del outs
        # 16-bit output: exactly RNE(float32 reference output) on every rank
        outs16 = comm.all_reduce_local(ts, cfg)
        want = ref32.to(tdt).view(torch.int16)
        for r in range(n):
            assert torch.equal(outs16[r].view(torch.int16), want), f"{tdt} output of rank {r}"
    finally:
        comm.close()
