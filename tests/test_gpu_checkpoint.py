"""On-disk formats of the device state: PBRLNET1 checkpoints
(net_pop.hpp:224-304) and serialize_state (algos.hpp:989-1015), byte-compatible with the
reference build (oracle/_ref, travels with the repo as a built .so)."""
import numpy as np
import pytest

from helpers import TD3_NETS, raw_at, to_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda):
    import paper_2206_08888_b200 as pb
    return pb


def _stepped(pb, ref, n, hidden, K, seed):
    from oracle.oracle import td3_defaults
    st = pb.make_td3_state(n, 17, 6, hidden, 1.0, seed, precision="ffma32")
    r = ref.td3(n, 17, 6, hidden, 1.0, seed)
    raw = ref.synthetic_batches(K, n, 32, 17, 6, seed)
    hy = pb.Td3Hyper.defaults(n)
    for k in range(K):
        pb.td3_update_step(st, to_batch(pb, raw, k), hy)
        r.step(raw_at(raw, k), td3_defaults(n))
    return st, r


def test_serialize_state_matches_reference_bytes(pb, ref, tmp_path):
    st, r = _stepped(pb, ref, 3, [32, 32], 4, 21)
    pb.serialize_state(st, tmp_path / "dev.bin")
    assert ref.lib.ref_td3f_serialize_state(r.h, str(tmp_path / "ref.bin").encode()) == 0
    a = (tmp_path / "dev.bin").read_bytes()
    b = (tmp_path / "ref.bin").read_bytes()
    assert len(a) == len(b) and a == b


def test_checkpoint_roundtrip_with_reference(pb, ref, tmp_path):
    st, r = _stepped(pb, ref, 2, [32, 32], 2, 5)
    for k, net in enumerate(TD3_NETS):
        # device -> reference
        p = tmp_path / f"dev_{net}.pbrl"
        pb.save_checkpoint(st, net, p)
        fresh = ref.td3(2, 17, 6, [32, 32], 1.0, 99)
        assert ref.lib.ref_td3f_load_checkpoint(fresh.h, k, str(p).encode()) == 0
        assert np.array_equal(fresh.get_net(net), st.params(net)), net
        # reference -> device
        q = tmp_path / f"ref_{net}.pbrl"
        assert ref.lib.ref_td3f_save_checkpoint(r.h, k, str(q).encode()) == 0
        assert p.read_bytes() == q.read_bytes()
        other = pb.make_td3_state(2, 17, 6, [32, 32], 1.0, 77, precision="bf16")
        pb.load_checkpoint(other, net, q)
        assert np.array_equal(other.params(net), r.get_net(net)), net


def test_load_checkpoint_rejects_mismatch(pb, tmp_path):
    a = pb.make_td3_state(2, 17, 6, [32, 32], 1.0, 1, precision="ffma32")
    b = pb.make_td3_state(3, 17, 6, [32, 32], 1.0, 1, precision="ffma32")
    p = tmp_path / "a.pbrl"
    pb.save_checkpoint(a, "policy", p)
    with pytest.raises(pb.ConfigError):
        pb.load_checkpoint(b, "policy", p)
    with pytest.raises(pb.ConfigError):
        pb.load_checkpoint(a, "critic1", p)
    bad = tmp_path / "bad.pbrl"
    bad.write_bytes(b"NOTPBRL!" + p.read_bytes()[8:])
    with pytest.raises(pb.ConfigError):
        pb.load_checkpoint(a, "policy", bad)
    trunc = tmp_path / "trunc.pbrl"
    trunc.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(pb.ConfigError):
        pb.load_checkpoint(a, "policy", trunc)


def test_replay_snapshot_matches_reference(pb, ref, tmp_path):
    """PBRLBUF1 (replay.hpp:113-165): device ring snapshots == the reference buffer's bytes
    (wrap-around included), and a reference snapshot loaded on the device samples identically."""
    n, ds, da, cap = 2, 17, 6, 40
    st = pb.make_td3_state(n, ds, da, [8], 1.0, 3)
    rep = pb.DeviceReplay(st, cap, "per_agent")
    rbufs = [ref.replay(cap, ds, da) for _ in range(n)]
    rng = np.random.default_rng(4)
    fills = [25, 95]
    mem = np.concatenate([np.full(f, m, np.uint32) for m, f in enumerate(fills)])
    rng.shuffle(mem)
    s, a = rng.standard_normal((mem.size, ds)), rng.standard_normal((mem.size, da))
    r, s2 = rng.standard_normal(mem.size), rng.standard_normal((mem.size, ds))
    d = (rng.random(mem.size) < 0.1).astype(np.float32)
    rep.insert(s, a, r, s2, d, mem)
    for i in range(mem.size):
        rbufs[mem[i]].push(s[i].astype(np.float32), a[i].astype(np.float32), float(r[i]),
                           s2[i].astype(np.float32), float(d[i]), int(mem[i]))
    for b in range(n):
        rep.save_snapshot(tmp_path / f"dev{b}.buf", b)
        assert ref.lib.ref_replay_save_snapshot(rbufs[b].h, str(tmp_path / f"ref{b}.buf").encode()) == 0
        assert (tmp_path / f"dev{b}.buf").read_bytes() == (tmp_path / f"ref{b}.buf").read_bytes()
    # reference snapshots -> a fresh device replay: same sampled batches as the original one
    st2 = pb.make_td3_state(n, ds, da, [8], 1.0, 3)
    rep2 = pb.DeviceReplay(st2, cap, "per_agent")
    for b in range(n):
        rep2.load_snapshot(tmp_path / f"ref{b}.buf", b)
        assert rep2.size(b) == rep.size(b)
    x = pb.sample_batch(rep, 64, seed=5, draw_id=3)
    y = pb.sample_batch(rep2, 64, seed=5, draw_id=3)
    for u, v in zip((x.s, x.a, x.r, x.s2, x.done), (y.s, y.a, y.r, y.s2, y.done)):
        assert np.array_equal(u, v)
    with pytest.raises(pb.ConfigError):
        pb.DeviceReplay(st2, cap + 1, "per_agent").load_snapshot(tmp_path / "ref0.buf", 0)


def test_deserialize_state_resumes_a_reference_run(pb, ref, tmp_path):
    """Full-trainer resume: the reference's serialize_state file of a run after K steps loads
    into a fresh device population, and K more steps on both leave bit-identical states."""
    from oracle.oracle import td3_defaults
    n, hidden, K, seed = 3, [32, 32], 3, 41
    r = ref.td3(n, 17, 6, hidden, 1.0, seed)
    raw = ref.synthetic_batches(2 * K, n, 32, 17, 6, seed)
    for k in range(K):  # odd K with delay 0.5: delay_acc = 0.5 at the cut
        r.step(raw_at(raw, k), td3_defaults(n))
    path = tmp_path / "ref_state.bin"
    assert ref.lib.ref_td3f_serialize_state(r.h, str(path).encode()) == 0
    st = pb.make_td3_state(n, 17, 6, hidden, 1.0, seed, precision="ffma32")
    pb.deserialize_state(st, path)
    hy = pb.Td3Hyper.defaults(n)
    for k in range(K, 2 * K):
        pb.td3_update_step(st, to_batch(pb, raw, k), hy)
        r.step(raw_at(raw, k), td3_defaults(n))
    for net in TD3_NETS:
        assert np.array_equal(st.params(net).view(np.uint32), r.get_net(net).view(np.uint32)), net
    pb.serialize_state(st, tmp_path / "dev.bin")
    assert ref.lib.ref_td3f_serialize_state(r.h, str(tmp_path / "ref2.bin").encode()) == 0
    assert (tmp_path / "dev.bin").read_bytes() == (tmp_path / "ref2.bin").read_bytes()


def test_deserialize_state_rejects_other_population(pb, tmp_path):
    a = pb.make_td3_state(2, 17, 6, [32, 32], 1.0, 1, precision="ffma32")
    b = pb.make_td3_state(3, 17, 6, [32, 32], 1.0, 1, precision="ffma32")
    pb.serialize_state(a, tmp_path / "a.bin")
    with pytest.raises(pb.ConfigError):
        pb.deserialize_state(b, tmp_path / "a.bin")
