"""The reference-side binding of INTEGRATION.md section 2
(integration/_kernels_b200.py) plugged into the UNMODIFIED reference package
(baseline/_ref, installed from /root/reference by pip --target): the
reference's own ``engine.execute`` and ``dense_attention_oracle`` run with
every block attention and merge computed by libtokenring on the GPU, at the
geometry of BASELINE config 1 (token ring, P=2, S=4096, H=8, D=64,
non-causal) and a causal zigzag case, against the reference's own numpy
backend on the same bf16-rounded inputs.

Skips when baseline/_ref is absent (it is git-ignored; bench/test boxes get
it with the repository snapshot)."""

import importlib
import importlib.util
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ringsim_b200():
    if not os.path.isdir(os.path.join(REF, "ringsim")):
        pytest.skip("baseline/_ref (the reference install) is absent")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    os.environ["RINGSIM_KERNELS"] = "python"          # the reference's numpy backend first
    ringsim = importlib.import_module("ringsim")
    kernels = importlib.import_module("ringsim.kernels")
    ref_impl = (kernels.attention_block, kernels.merge_state)
    # what the maintainer's one-line branch in ringsim/kernels.py does
    spec = importlib.util.spec_from_file_location(
        "ringsim._kernels_b200", os.path.join(ROOT, "integration", "_kernels_b200.py"))
    b200 = importlib.util.module_from_spec(spec)
    sys.modules["ringsim._kernels_b200"] = b200
    spec.loader.exec_module(b200)
    yield ringsim, kernels, b200, ref_impl
    kernels.attention_block, kernels.merge_state = ref_impl


def _bf16(x):
    import torch
    return torch.as_tensor(x).to(torch.float32).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("kind,P,S,H,D,causal", [
    ("token-ring", 2, 4096, 8, 64, False),           # BASELINE config 1 geometry
    ("zigzag-token-ring", 4, 2048, 2, 128, True)])
def test_reference_execute_on_b200_backend(ringsim_b200, kind, P, S, H, D, causal):
    ringsim, kernels, b200, (ref_attn, ref_merge) = ringsim_b200
    from ringsim import engine, rng
    q, k, v = (_bf16(x) for x in rng.attention_inputs(0, S, H, D))
    sched = (engine.build_token_ring(P, S, H, D) if kind == "token-ring"
             else engine.build_zigzag_token_ring(P, S, H, D))
    kernels.attention_block, kernels.merge_state = ref_attn, ref_merge
    want, _ = engine.execute(sched, q, k, v)
    kernels.attention_block, kernels.merge_state = b200.attention_block, b200.merge_state
    assert kernels.attention_block is b200.attention_block
    got, trace = engine.execute(sched, q, k, v)
    for r in range(P):
        assert np.abs(got[r].out - want[r].out).max() <= 2e-2, r
        assert np.abs(got[r].lse - want[r].lse).max() <= 1e-3, r
    # the reference's own oracle and error metric, with the B200 backend underneath
    full = ringsim.global_reorder(got, sched.partition)
    dense = ringsim.dense_attention_oracle(q, k, v, causal=causal)
    kernels.attention_block, kernels.merge_state = ref_attn, ref_merge
    dense_ref = ringsim.dense_attention_oracle(q, k, v, causal=causal)
    assert np.abs(dense.out - dense_ref.out).max() <= 2e-2
    assert ringsim.max_relative_error(full, dense_ref) <= 2e-2
