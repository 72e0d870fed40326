"""Host-side call order of ShiftStep.run (no GPU): where the caller's collective lands
relative to the shift backward and the join of the preprocess's SH-coefficient stream
(step.py; bench.py passes the shift payload's all_reduce with collective_after_sh=False,
the full payload with True).  The kernels are replaced by recorders."""
import types

import pytest

from paper_2411_14847_b200 import step as step_mod


class FakePass:
    def __init__(self, log):
        self.log, self.defer_sh, self.uv_out = log, False, None

    def run(self, sh, rec, dLs, g, project=None):
        self.log.append(("pass", self.defer_sh))

    def join_sh(self):
        self.log.append(("join_sh",))


class FakeGrads:
    uv = None
    pos_opa = rot = g_mu = g_sigma = flat = None

    def zero_(self):
        pass


def make_step(log, shift=True):
    st = step_mod.ShiftStep.__new__(step_mod.ShiftStep)
    st.cams, st.deg, st.shift, st.validate = [object()], 3, shift, False
    st.split = [-1]
    st.records = types.SimpleNamespace()
    st.mvp = FakePass(log)
    st._errmap_pos = None
    return st


def bufs():
    base = types.SimpleNamespace(pos_opa=None, rot=None, dynamic=None)
    return types.SimpleNamespace(grads=FakeGrads(), base=base, mu=None, sigma=None, dLs=None,
                                 shifted=types.SimpleNamespace(pos_opa=None, rot=None))


@pytest.fixture
def log(monkeypatch):
    log = []
    fake = types.SimpleNamespace(
        dass_apply_shift=lambda *a: log.append(("shift",)),
        dass_apply_shift_bwd=lambda *a: log.append(("shift_bwd",)),
        DASS_PROJECT_ALL=0)
    monkeypatch.setattr(step_mod, "dass", fake)
    return log


@pytest.mark.parametrize("after_sh,expect", [
    (False, [("shift",), ("pass", True), ("shift_bwd",), ("coll",), ("join_sh",)]),
    (True, [("shift",), ("pass", False), ("shift_bwd",), ("join_sh",), ("coll",)]),
], ids=["shift_payload_early", "full_payload_after_join"])
def test_collective_position(log, after_sh, expect):
    st = make_step(log)
    st.run(bufs(), collective=lambda: log.append(("coll",)), collective_after_sh=after_sh)
    assert log == expect
    assert st.mvp.defer_sh is False      # the deferral does not leak into the next call


def test_no_collective_joins_before_returning(log):
    st = make_step(log)
    st.run(bufs())
    assert log == [("shift",), ("pass", False), ("shift_bwd",), ("join_sh",)]


def test_plain_step_without_shift(log):
    st = make_step(log, shift=False)
    st.run(bufs(), collective=lambda: log.append(("coll",)), collective_after_sh=False)
    assert log == [("pass", True), ("coll",), ("join_sh",)]
