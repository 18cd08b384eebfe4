"""Snapshot publication: SnapshotMailbox / ActorSnapshot
(pipeline.hpp:31-83) and actor_loop's refresh (pipeline.hpp:255-285), device-resident.  An actor
holds its own population handle and acts on the snapshot it adopted while the learner keeps
updating; no torn snapshot is ever observed under concurrency."""
import threading

import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _fnv(data: bytes, h: int) -> int:
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _checksum(params, dims, explore):
    """ActorSnapshot::compute_checksum (pipeline.hpp:38-47) from flatten_member rows: every
    layer's weights of all members [N][in][out], then its biases, then explore_std."""
    h = 1469598103934665603
    off = 0
    for i, o in zip(dims[:-1], dims[1:]):
        h = _fnv(np.ascontiguousarray(params[:, off:off + i * o]).tobytes(), h)
        h = _fnv(np.ascontiguousarray(params[:, off + i * o:off + i * o + o]).tobytes(), h)
        off += i * o + o
    return _fnv(np.asarray(explore, np.float64).tobytes(), h)


@pytest.mark.parametrize("precision", ["ffma32", "bf16"])
def test_actor_acts_on_the_published_snapshot(pb, precision):
    n, ds, da = 4, 17, 6
    learner = pb.make_td3_state(n, ds, da, [64, 64], 1.0, 3, precision=precision)
    actor = pb.make_td3_state(n, ds, da, [64, 64], 1.0, 99, precision=precision)
    mb = pb.SnapshotMailbox(learner)
    assert mb.version() == 0 and pb.actor_refresh(actor, mb)[0] == 0
    explore = [0.1, 0.2, 0.3, 0.4]
    assert mb.publish(learner, explore) == 1
    v, ex = pb.actor_refresh(actor, mb)
    assert v == 1 and ex.tolist() == explore
    assert bits_equal(actor.params("policy"), learner.params("policy"))
    obs = np.random.default_rng(0).uniform(-1, 1, (n, 7, ds)).astype(np.float32)
    steps = np.arange(n, dtype=np.uint64)
    a0 = pb.act(learner, obs, explore, 5, steps, True)
    assert np.array_equal(pb.act(actor, obs, ex, 5, steps, True), a0)
    # the learner moves on; the actor keeps its snapshot until the next publish + refresh
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [1.0] * n
    for b in pb.make_synthetic_batches(3, n, 64, ds, da, 4):
        pb.td3_update_step(learner, b, hy)
    assert pb.actor_refresh(actor, mb)[0] == 1
    assert np.array_equal(pb.act(actor, obs, ex, 5, steps, True), a0)
    assert mb.publish(learner, explore) == 2
    assert pb.actor_refresh(actor, mb)[0] == 2
    assert np.array_equal(pb.act(actor, obs, ex, 5, steps, True),
                          pb.act(learner, obs, explore, 5, steps, True))
    ver, cs = mb.checksum()
    assert ver == 2
    assert cs == _checksum(learner.params("policy"), [ds, 64, 64, da], explore)


def test_concurrent_publish_and_refresh_never_tears(pb):
    """Learner thread: update + publish in a loop; actor thread: refresh + act.  Every action
    block the actor produced must equal the actions of exactly the snapshot version it held."""
    n, ds, da = 3, 11, 3
    learner = pb.make_td3_state(n, ds, da, [64, 64], 1.0, 8)
    actor = pb.make_td3_state(n, ds, da, [64, 64], 1.0, 8)
    mb = pb.SnapshotMailbox(learner)
    hy = pb.Td3Hyper.defaults(n)
    hy.policy_delay_ratio = [1.0] * n
    batches = pb.make_synthetic_batches(4, n, 32, ds, da, 9)
    obs = np.random.default_rng(1).uniform(-1, 1, (n, 5, ds)).astype(np.float32)
    steps = np.zeros(n, np.uint64)
    published = {}
    seen = []
    stop = threading.Event()

    def actor_loop():
        while not stop.is_set() or len(seen) < 3:
            v, ex = pb.actor_refresh(actor, mb)
            if v:
                seen.append((v, pb.act(actor, obs, ex, 1, steps, True)))

    published[mb.publish(learner, [0.1] * n)] = learner.params("policy")
    t = threading.Thread(target=actor_loop)
    t.start()
    try:
        for i in range(12):
            pb.td3_update_step(learner, batches[i % 4], hy)
            published[mb.publish(learner, [0.1] * n)] = learner.params("policy")
    finally:
        stop.set()
        t.join(timeout=120)
    assert seen and [v for v, _ in seen] == sorted(v for v, _ in seen)
    checker = pb.make_td3_state(n, ds, da, [64, 64], 1.0, 8)
    for v in sorted({v for v, _ in seen}):
        for m in range(n):
            checker.unflatten_member("policy", m, published[v][m])
        want = pb.act(checker, obs, [0.1] * n, 1, steps, True)
        for vv, got in seen:
            if vv == v:
                assert np.array_equal(got, want), v
