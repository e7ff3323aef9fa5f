"""Host-side plan policies (no GPU): protocol choice, counter-release mode,
window-major execution, L2 hints and chunk-group split, read from the plan
summary of host-only plans (device=-1).  The thresholds are the measured
ones documented in DESIGN.md section 4."""
import pytest

from paper_2008_08708_b200 import sccl
from paper_2008_08708_b200 import schedules as S

P = 8
AG = S.hamiltonian_allgather(P)
SCHED = {
    "ag777": (S.to_json(AG), sccl.U8),
    "ring": (S.to_json(S.ring_allgather(P)), sccl.U8),
    "ag111": (S.to_json(S.one_shot_allgather(P)), sccl.U8),
    "a2a": (S.to_json(S.direct_alltoall(P)), sccl.U8),
    "ar822": (S.allreduce_from(S.one_shot_allgather(P)), sccl.BF16),
    "ar56": (S.allreduce_from(AG), sccl.BF16),
}


def info(name, nbytes, **kw):
    js, dt = SCHED[name]
    plan = sccl.LoopbackPlan(js, nbytes, dt, device=-1, **kw)
    try:
        return plan.info()
    finally:
        plan.close()


@pytest.mark.parametrize("name", list(SCHED))
def test_small_is_ll_large_is_simple(name):
    assert info(name, 1024)["protocol"] == "ll"
    assert info(name, 64 << 20)["protocol"] == "simple"


def test_window_major_only_for_streaming_relay_schedules():
    # relays / reductions re-read receipts: window-major above 1 GB per launch
    for name in ("ag777", "ring", "ar56"):
        assert info(name, 128 << 20, protocol="simple")["window"] > 0, name
        assert info(name, 4 << 20, protocol="simple")["window"] == 0, name
    assert info("ar822", 128 << 20, protocol="simple", pull="off")["window"] > 0
    # nothing is re-read: op-major at any size (the pull-lowered one-shot
    # allreduce reads peers' inputs in place, it has no receipts to re-read)
    for name in ("ag111", "a2a", "ar822"):
        assert info(name, 128 << 20, protocol="simple")["window"] == 0, name


def test_window_size_follows_ops_per_step():
    ring = info("ring", 128 << 20, protocol="simple")  # one op per step: 4 tiles
    assert ring["window"] == 4 * ring["tile_bytes"]
    ar56 = info("ar56", 128 << 20, protocol="simple")  # seven ops per step: 1 tile
    assert ar56["window"] == ar56["tile_bytes"]


def test_no_chunk_group_split_for_big_copy_relays():
    # round 2: one chunk group beat the round-1 two-group split at 64-512 MiB
    # (profiles/r02/s2_ag_split_ab.jsonl); the split stays as a policy-table
    # flag (group_split) for SCCL_POLICY overrides
    big = info("ag777", 128 << 20, protocol="simple")
    assert big["chunk_groups"] == 1 and big["window"] == big["tile_bytes"]
    assert info("ag777", 16 << 20, protocol="simple")["chunk_groups"] == 1
    assert info("ar56", 128 << 20, protocol="simple")["chunk_groups"] == 1


@pytest.mark.parametrize("mb,tile", [(1, 32768), (4, 32768), (8, 65536), (12, 65536), (16, 16384), (48, 16384),
                                     (64, 32768), (128, 32768)])
def test_pulled_one_shot_allreduce_tiles(mb, tile):
    # round 2: 32 KiB tiles up to 512 KiB chunks (session 3,
    # profiles/r02/s3_ar822_mid.jsonl; 16 KiB before) and 16 KiB from 250 MB
    # of program traffic to the streaming threshold (profiles/r02/s2_ar822_tile.jsonl)
    assert info("ar822", mb << 20, protocol="simple")["tile_bytes"] == tile
    if mb == 4:  # push-lowered (multi-process style) keeps the round-1 rule
        assert info("ar822", mb << 20, protocol="simple", pull="off")["tile_bytes"] == 65536


def test_simple_chunk_groups_follow_the_chunks_a_rank_works_on():
    # round 2: one-shot copies / pulled one-shot reductions have one chunk of
    # work per rank in the simple protocol; the CTAs go to byte parts
    # (profiles/r02/s2_workchunks_ab.jsonl)
    i = info("ag111", 64 << 10, protocol="simple")
    assert (i["chunk_groups"], i["byte_parts"]) == (1, 8)
    i = info("ar822", 1 << 20, protocol="simple")
    assert (i["chunk_groups"], i["byte_parts"]) == (1, 16)
    assert info("a2a", 256 << 10, protocol="simple")["chunk_groups"] == 8  # 8 chunks of work per rank
    assert info("ag111", 1 << 10, protocol="ll")["chunk_groups"] == 8      # LL unpacks receipts in ops: unchanged
    js, dt = SCHED["ag111"]  # one rank per GPU: the same cap (32 CTAs per rank, all on the rank's chunk)
    mp = sccl.Plan(js, 0, P, 256 << 10, dt, device=-1, protocol="simple")
    try:
        i = mp.info()
    finally:
        mp.close()
    assert (i["chunk_groups"], i["byte_parts"]) == (1, 32)


def test_l2_hints_above_one_gigabyte():
    assert info("ag777", 128 << 20, protocol="simple")["l2hint"] == 1
    assert info("a2a", 128 << 20, protocol="simple")["l2hint"] == 1
    assert info("ar822", 128 << 20, protocol="simple")["l2hint"] == 0  # pulled one-shot: faster without (round 2)
    assert info("ar822", 128 << 20, protocol="simple", pull="off")["l2hint"] == 1
    assert info("ar822", 16 << 20, protocol="simple")["l2hint"] == 0
    assert info("ag777", 1 << 20, protocol="simple")["l2hint"] == 0


def test_relays_evict_last_only_when_discarded():
    assert info("ag777", 128 << 20, protocol="simple")["relay_evict_last"] == 0
    assert info("ar56", 128 << 20, protocol="simple")["relay_evict_last"] == 1  # its receipts are discarded
    assert info("ar822", 128 << 20, protocol="simple", pull="off")["relay_evict_last"] == 1  # discarded after use
    assert info("ar822", 16 << 20, protocol="simple")["relay_evict_last"] == 0   # no hints at all


def test_discard_only_for_wide_streaming_reductions():
    assert info("ar822", 128 << 20, protocol="simple", pull="off")["discard"] == 1   # fan-in 8
    assert info("ar822", 128 << 20, protocol="simple")["discard"] == 0   # pull: no receipts
    assert info("ar56", 128 << 20, protocol="simple")["discard"] == 1    # 2-input reduce chain (round 2)
    assert info("ar822", 16 << 20, protocol="simple")["discard"] == 0    # fits L2
    assert info("ag777", 128 << 20, protocol="simple")["discard"] == 0   # no reduction


def test_counter_release_mode():
    assert info("ring", 1 << 20, protocol="simple")["selfpub"] == 1   # <= 16 tiles per CTA
    assert info("ag777", 128 << 20, protocol="simple")["selfpub"] == 0


def test_env_overrides(monkeypatch):
    monkeypatch.setenv("SCCL_WINDOW", "0")
    monkeypatch.setenv("SCCL_L2HINT", "0")
    monkeypatch.setenv("SCCL_SELFPUB", "1")
    i = info("ag777", 128 << 20, protocol="simple")
    assert i["window"] == 0 and i["l2hint"] == 0 and i["selfpub"] == 1
    monkeypatch.setenv("SCCL_WINDOW", "4096")
    assert info("ag111", 1 << 20, protocol="simple")["window"] == 4096


def test_multiprocess_plans_use_the_sys_scope_model():
    """One rank per GPU signals at system scope: the bulk step is dearer, so
    the LL protocol is chosen up to larger sizes than in loopback."""
    js, dt = SCHED["ring"]
    sizes = [1 << k for k in range(12, 25)]

    def last_ll(make):
        best = 0
        for sz in sizes:
            plan = make(sz)
            if plan.info()["protocol"] == "ll":
                best = sz
            plan.close()
        return best

    loop = last_ll(lambda sz: sccl.LoopbackPlan(js, sz, dt, device=-1))
    multi = last_ll(lambda sz: sccl.Plan(js, 0, P, sz, dt, device=-1))
    assert multi >= loop > 0


def test_chunk_groups_balanced_only_when_modulo_is_lopsided():
    # alltoall chunk ids are i*P + rank: with kc = 2 every rank's ops would
    # share one group under chunk % kc
    assert info("a2a", 4 << 20, protocol="simple")["groups_balanced"] == 1
    assert info("ag777", 128 << 20, protocol="simple")["groups_balanced"] == 0  # within 25 % of the mean


def test_ll_chains_run_one_chunk_per_cta():
    # >= 4 steps, >= 32 chunks of <= 40 KiB: kc = G, kb = 1
    i = info("ag777", 64 << 10, protocol="ll")
    assert (i["chunk_groups"], i["byte_parts"]) == (56, 1)
    i = info("ar56", 1 << 20, protocol="ll")
    assert (i["chunk_groups"], i["byte_parts"]) == (56, 1)
    # single-step alltoall keeps byte parts
    assert info("a2a", 256 << 10, protocol="ll")["byte_parts"] > 1


def test_ll_splits_chunks_when_groups_run_out():
    # one-shot allreduce: 8 chunk groups only; 64 KiB -> 8 KiB chunks in 2 KiB parts
    i = info("ar822", 64 << 10, protocol="ll")
    assert (i["chunk_groups"], i["byte_parts"]) == (8, 4)


def test_multiprocess_plans_do_not_inherit_loopback_hbm_policies():
    """One rank per GPU: NVLink, not the shared HBM, is the bound, so the
    loopback-tuned streaming policies stay off (policy.hpp): no window-major
    order, no L2 hints, no receipt discards, no chunk-group split, at most 32
    CTAs per rank; the plan reports its table's version."""
    for name, nb in (("ag777", 128 << 20), ("ar822", 512 << 20), ("ar56", 512 << 20), ("ring", 1 << 30)):
        js, dt = SCHED[name]
        mp = sccl.Plan(js, 0, P, nb, dt, device=-1, protocol="simple").info()
        assert mp["policy"].startswith("multiprocess"), mp["policy"]
        assert (mp["window"], mp["l2hint"], mp["discard"]) == (0, 0, 0), (name, mp)
        assert mp["chunk_groups"] * mp["byte_parts"] <= 32 and mp["chunk_groups"] == 1, (name, mp)
        lb = info(name, nb, protocol="simple")
        assert lb["policy"].startswith("loopback")
    assert info("ag777", 128 << 20, protocol="simple")["window"] > 0  # the loopback table keeps them


def test_policy_table_override(tmp_path):
    """SCCL_POLICY replaces a table at run time (tools/tune.py --multi writes
    one from an N>1 sweep); read once per process."""
    import json
    import subprocess
    import sys
    t = tmp_path / "policy.json"
    t.write_text(json.dumps({"multiprocess": {"version": "multiprocess-test", "window_major": True,
                                              "l2_hints": True, "max_ctas_per_rank": 8,
                                              "simple_alpha": 100.0},
                             "loopback": {"version": "loopback-test", "group_split": True}}))
    code = ("import sys, json; sys.path.insert(0, %r)\n"
            "from paper_2008_08708_b200 import sccl, schedules as S\n"
            "js = S.to_json(S.hamiltonian_allgather(8))\n"
            "i = sccl.Plan(js, 0, 8, 128 << 20, sccl.U8, device=-1, protocol='simple').info()\n"
            "j = sccl.Plan(js, 0, 8, 1 << 20, sccl.U8, device=-1).info()\n"
            "k = sccl.LoopbackPlan(js, 128 << 20, sccl.U8, device=-1, protocol='simple').info()\n"
            "print(json.dumps([i['policy'], i['window'] > 0, i['l2hint'], i['nchannels'], j['protocol'],\n"
            "                  k['policy'], k['chunk_groups']]))"
            % str(sccl._HERE.rsplit("/", 1)[0]))
    out = subprocess.run([sys.executable, "-c", code], env={**__import__("os").environ, "SCCL_POLICY": str(t)},
                         capture_output=True, text=True, check=True).stdout
    pol, window, l2, nch, proto, lpol, kc = json.loads(out)
    assert pol == "multiprocess-test" and window and l2 == 1 and nch <= 8
    assert proto == "ll"  # a 100 us bulk step makes LL win at 1 MiB
    assert lpol == "loopback-test" and kc == 2  # the round-1 chunk-group split, back on by table
