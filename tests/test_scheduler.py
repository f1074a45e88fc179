"""Host-side scheduler (the GPU path's caller): reference policy properties + decode-priority policy."""

import math

import numpy as np
import pytest

from paper_2512_02281_b200.scheduler import (
    ControlGains,
    FeedbackSample,
    QueueEntry,
    SchedulerConfig,
    TwoQueueScheduler,
    slack,
)


def pre(rid, t, ddl, est=0.0):
    return QueueEntry(request_id=rid, stage="prefill", t_arrival=t, deadline=ddl, est_remaining_extends=est)


def dec(rid, t):
    return QueueEntry(request_id=rid, stage="decode", t_arrival=t)


def test_slack_known_answers():  # scheduler.py:129-133 (acceptance criterion 5 values)
    assert slack(pre(0, 0.0, 100.0, 5.0), 40.0, 2.0) == 50.0
    assert slack(pre(0, 0.0, 100.0, 0.0), 70.0, 3.0) == 30.0
    assert slack(pre(0, 0.0, 10.0, 1.0), 20.0, 5.0) == -15.0
    with pytest.raises(ValueError):
        slack(dec(0, 0.0), 0.0, 1.0)


def test_entry_validation():
    with pytest.raises(ValueError):
        QueueEntry(request_id=0, stage="prefill", t_arrival=1.0)
    with pytest.raises(ValueError):
        pre(0, 2.0, 1.0)
    with pytest.raises(ValueError):
        QueueEntry(request_id=0, stage="other", t_arrival=0.0)


def test_reservation_and_give_back():
    s = TwoQueueScheduler(SchedulerConfig(slots_n=8, r=0.25))
    assert s.reservation() == 2
    for i in range(5):
        s.enqueue(pre(i, 0.0, 10.0))
    plan = s.build_batch(1.0)  # no decode: prefill takes every slot it can
    assert (plan.n_pre, plan.n_dec, plan.pad_count) == (5, 0, 3)
    for i in range(10):
        s.enqueue(dec(100 + i, float(i)))
    s.enqueue(pre(9, 0.0, 10.0))
    plan = s.build_batch(1.0)
    assert (plan.n_pre, plan.n_dec) == (1, 7)


def test_orders_and_invariants_random_states():  # acceptance criterion 4 property, 2000 states
    rng = np.random.Generator(np.random.Philox(20_240_605))
    for _ in range(2000):
        n = int(rng.integers(1, 17))
        r_min = float(rng.uniform(0.0, 0.4))
        r_max = float(rng.uniform(r_min, 1.0))
        r = float(rng.uniform(r_min, r_max))
        s = TwoQueueScheduler(SchedulerConfig(slots_n=n, r=r, r_min=r_min, r_max=r_max))
        t_now = float(rng.uniform(0, 100))
        n_pre, n_dec = int(rng.integers(0, 3 * n)), int(rng.integers(0, 3 * n))
        for i in range(n_pre):
            a = float(rng.uniform(0, t_now))
            s.enqueue(pre(i, a, a + float(rng.uniform(0, 50)), float(rng.uniform(0, 20))))
        for i, a in enumerate(sorted(float(rng.uniform(0, t_now)) for _ in range(n_dec))):
            s.enqueue(dec(1000 + i, a))
        s.t_ext = float(rng.uniform(0.1, 5.0))
        resv = s.reservation()
        plan = s.build_batch(t_now)
        assert plan.n_pre + plan.n_dec + plan.pad_count == n
        if n_pre >= resv:
            assert plan.n_pre >= resv
        sl = [slack(e, t_now, s.t_ext) for e in plan.picked_prefill]
        assert sl == sorted(sl)
        if sl and s.q_pre:
            assert min(slack(e, t_now, s.t_ext) for e in s.q_pre) >= sl[-1]
        arr = [e.t_arrival for e in plan.picked_decode]
        assert arr == sorted(arr)
        if arr and s.q_dec:
            assert min(e.t_arrival for e in s.q_dec) >= arr[-1]


def test_should_launch_rules():
    s = TwoQueueScheduler(SchedulerConfig(slots_n=4, tau_pre=1.0, tau_global=3.0))
    s.enqueue(dec(0, 0.0))
    assert not s.should_launch(2.0)
    assert s.should_launch(3.0)  # global timeout
    s.enqueue(pre(1, 2.5, 10.0))
    assert s.should_launch(3.5)  # aged prefill (and global)
    for i in range(4):
        s.enqueue(dec(10 + i, 3.6))
    assert s.should_launch(3.6)  # full buffer


def test_control_loop_response():  # acceptance criterion 6
    gains = ControlGains(interval=1.0, delta_r=0.0625, beta_tau=0.5, tau_pre_min=0.25)
    cfg = SchedulerConfig(r=0.25, r_min=0.25, r_max=0.75, tau_pre=2.0, tau_global=10.0, control=gains)
    s = TwoQueueScheduler(cfg)
    want = math.ceil((cfg.r_max - cfg.r_min) / gains.delta_r)
    reached = None
    for i in range(20):
        r, _ = s.control_update(FeedbackSample(0.0, 0.5, 0.0, 0.0))
        if reached is None and r == cfg.r_max:
            reached = i + 1
    assert reached == want and s.tau_pre == gains.tau_pre_min
    for _ in range(20):
        s.control_update(FeedbackSample(0.0, 0.95, 0.0, 0.8))
    assert s.r == cfg.r_min


def test_ema():
    s = TwoQueueScheduler(SchedulerConfig(t_ext_ema_gamma=0.5))
    assert s.record_extend_latency(2.0) == 2.0
    assert s.record_extend_latency(4.0) == 3.0
    with pytest.raises(ValueError):
        s.record_extend_latency(0.0)


def test_decode_priority_serves_decode_first():
    s = TwoQueueScheduler(SchedulerConfig(slots_n=4, policy="decode_priority", min_prefill=1))
    for i in range(3):
        s.enqueue(pre(i, 0.0, 100.0))
    for i in range(3):
        s.enqueue(dec(10 + i, float(i)))
    plan = s.build_batch(1.0)
    assert [e.request_id for e in plan.picked_decode] == [10, 11, 12]
    assert plan.n_pre == 1  # leftover slot only
    # a late prefill keeps its guaranteed slot even under decode pressure
    s2 = TwoQueueScheduler(SchedulerConfig(slots_n=4, policy="decode_priority", min_prefill=1))
    s2.enqueue(pre(0, 0.0, 1.0))
    for i in range(8):
        s2.enqueue(dec(10 + i, float(i)))
    plan = s2.build_batch(5.0)
    assert plan.n_pre == 1 and plan.n_dec == 3


def test_decode_priority_preempts_planned_prefill():
    s = TwoQueueScheduler(SchedulerConfig(slots_n=4, policy="decode_priority", min_prefill=1))
    for i in range(4):
        s.enqueue(pre(i, 0.0, 100.0))
    plan = s.build_batch(1.0)
    assert plan.n_pre == 4
    s.enqueue(dec(50, 1.5))
    s.enqueue(dec(51, 1.6))
    plan = s.preempt(plan, 2.0)
    assert plan.n_dec == 2 and plan.n_pre == 2 and len(s.q_pre) == 2
    assert plan.n_pre + plan.n_dec + plan.pad_count == 4


def test_config_validation():
    with pytest.raises(ValueError):
        SchedulerConfig(policy="fifo")
    with pytest.raises(ValueError):
        SchedulerConfig(tau_pre=5.0, tau_global=1.0)
    with pytest.raises(ValueError):
        SchedulerConfig(r=0.9, r_max=0.5)
