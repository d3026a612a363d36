"""GPU: every stage kernel is bitwise deterministic at a size with enough CTAs per
SM to expose pipeline races (the stage-release WAR race of the mbarrier ring was
only visible from ~2e5 CTAs on), and repeated steps reproduce bitwise
(test_stepper.cpp:323-332)."""
import ctypes as C

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from paper_2601_06849_b200 import configs

pytestmark = pytest.mark.gpu

STAGES_L1 = ["z_fwd", "z_back", "y_fwd", "y_back", "x_fwd_mix", "x_back_src", "x_fwd_corr", "x_back_upd"]
STAGES_L2_R01 = [f"{s}_{h}" for s in ["z_fwd_even", "z_fwd_odd", "z_back_o", "z_back_e", "y_fwd_even", "y_fwd_odd",
                                       "y_back_o", "y_back_e", "x_fwd_mix_even", "x_fwd_mix_odd"] for h in "ab"] + \
                ["x_back_src_o", "x_back_src_e", "x_fwd_corr_even", "x_fwd_corr_odd", "x_back_upd_o", "x_back_upd_e"]
# default level 2: every backward transform is one fused launch (etd_back6)
# (the y/z ones one field per launch: S = 1 tiles, XPAIR fragment interleave)
STAGES_L2 = ["z_fwd_even_a", "z_fwd_even_b", "z_fwd_odd_a", "z_fwd_odd_b", "z_back_a", "z_back_b", "z_back_c", "z_back_d",
             "y_fwd_even_a", "y_fwd_even_b", "y_fwd_odd_a", "y_fwd_odd_b", "y_back_a", "y_back_b", "y_back_c", "y_back_d",
             "x_fwd_mix_even_a", "x_fwd_mix_even_b", "x_fwd_mix_odd_a", "x_fwd_mix_odd_b", "x_back_src",
             "x_fwd_corr_even", "x_fwd_corr_odd", "x_back_upd"]


@pytest.mark.parametrize("level", ["1", "2", "2-r01"])
def test_stage_kernels_are_deterministic(level, monkeypatch):
    if level == "1":
        monkeypatch.setenv("ETD_FOLD2", "0")
    if level == "2-r01":
        monkeypatch.setenv("ETD_BACK6", "0")
    cfg = configs.CONFIGS[4]
    n = 383
    plan = configs.make_plan(cfg, n)
    assert plan.fold_level() == (int(level[0]),) * 3
    stages = {"1": STAGES_L1, "2": STAGES_L2, "2-r01": STAGES_L2_R01}[level]
    assert [s["name"] for s in plan.stage_stats() if s["flops_per_launch"] > 0] == stages
    for s, a in enumerate(configs.initial_state(cfg, n)):
        plan.upload(s, a)
    plan.step(1)
    L = etd.lib()
    L.etd_debug_repeat_op.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_longlong),
                                      C.c_void_p, C.c_int]
    for name in stages:
        # the y/z fused backward launches hold one field each, every other launch two
        for out in ((0,) if level == "2" and name[:6] in ("z_back", "y_back") else (0, 1)):
            mm = C.c_longlong(-1)
            rc = L.etd_debug_repeat_op(plan.handle, name.encode(), out, 6, C.byref(mm), None, 0)
            assert rc == 0 and mm.value == 0, (name, out, mm.value)


def test_repeated_full_size_like_steps_bitwise():
    cfg = configs.CONFIGS[3]
    n = 255
    ics = configs.initial_state(cfg, n)
    res = []
    for _ in range(2):
        plan = configs.make_plan(cfg, n)
        st = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, *ics), cfg.source, nsteps=2)
        plan.upload(0, ics[0])
        plan.upload(1, ics[1])
        plan.step(2)
        u, _, _ = plan.download(0)
        assert np.array_equal(u, st.U)  # pipelined == resident
        res.append(st.U)
        plan.close()
    assert np.array_equal(res[0], res[1])
