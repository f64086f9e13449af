"""Reyes Split/Dice/Sample/Shade on the GPU
against the oracle: the diced micropolygon mesh bit-exact (positions, normals,
indices), the frame and the 32x32-bin lists bit-exact, RGB within 1e-5."""
from __future__ import annotations

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(oracle_lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1404_6293_b200 as piko
    return piko, oracle_lib, torch


@pytest.mark.parametrize("name", ["small", "c6"])
@pytest.mark.parametrize("bw", [32, 16])
def test_reyes_dice_and_sample_match_oracle(env, name, bw):
    piko, orc, torch = env
    s = scenes.scene_patches(n=4, seed=61, dice_px=3.0, name="small") if name == "small" else scenes.scene_c6()
    dev = torch.device("cuda:0")
    pt = torch.from_numpy(s.patches).to(dev)
    r = piko.Renderer(s.W, s.H, bw, device=dev)
    piko.piko_set_debug(r.ctx, piko.PIKO_DEBUG_COVERAGE_COUNT)
    r.draw_patches(pt, s.mvp, s.light, s.dice_px, s.max_grid)
    torch.cuda.synchronize()
    G, ov, oi = orc.dice(s.patches, s.mvp, s.W, s.H, s.dice_px, s.max_grid)
    gv, gi = r.diced()
    gv, gi = gv.cpu().numpy(), gi.cpu().numpy()
    assert gv.shape == ov.shape and gi.shape == oi.shape
    assert np.array_equal(gv.view(np.uint32), ov.view(np.uint32)), "diced vertices differ"
    assert np.array_equal(gi, oi), "diced indices differ"
    ref = orc.render(ov, oi, s.mvp, s.light, s.W, s.H, want_covcount=True)
    assert np.array_equal(r.primid().cpu().numpy(), ref["primid"])
    assert np.array_equal(r.depth.cpu().numpy().view(np.uint32), ref["depth"].view(np.uint32))
    assert np.array_equal(r.coverage().cpu().numpy().view(np.uint32), ref["covcount"])
    assert np.abs(r.rgba.cpu().numpy() - ref["rgba"]).max() <= 1e-5
    st, pr = r.bins()
    ost, opr = orc.bins(ov, oi, s.mvp, s.W, s.H, bw, bw)
    assert np.array_equal(st.cpu().numpy(), ost) and np.array_equal(pr.cpu().numpy(), opr)
    r.close()


def test_reyes_argument_validation(env):
    piko, _, torch = env
    s = scenes.scene_patches(n=2, seed=62, name="tiny")
    pt = torch.from_numpy(s.patches).cuda()
    r = piko.Renderer(s.W, s.H, 32)
    for dp, mg in ((0.0, 64), (float("nan"), 64), (1.0, 3), (1.0, 0), (1.0, 2048)):
        assert r.draw_patches(pt, s.mvp, s.light, dp, mg, check=False) == piko.PIKO_EINVAL
    assert r.draw_patches(pt[:0], s.mvp, s.light, 2.0, 64, check=False) == piko.PIKO_OK  # no patches: clear
    torch.cuda.synchronize()
    assert (r.primid().cpu().numpy() == -1).all()
    r.close()
