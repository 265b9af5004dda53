"""Generate golden vectors by running the REAL reference (`sessiondedup`).

Run in the build container (where `/root/reference` exists):

    python tests/golden/make_golden.py

Writes `tests/golden/{dedup,pool,jagged,slice,datagen,errors,transforms,wire,partial,sdd}.npz`.  These
fixtures pin the oracle restatement (`oracle/`) and the CUDA path; the GPU box
never needs `/root/reference`.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from sessiondedup import tensors as T  # noqa: E402
from sessiondedup import trainer_sim as TS  # noqa: E402
from sessiondedup import datagen as DG  # noqa: E402
from sessiondedup import reader as RD  # noqa: E402

OUT = Path(__file__).resolve().parent


def _kjt(rows, keys):
    kjt = T.build_kjt(rows, keys)
    return [(np.array(kjt.entries[k].values), np.array(kjt.entries[k].offsets)) for k in keys]


def _store_case(store, name, keys, rows):
    ik = T.build_ikjt(rows, keys)
    feats = _kjt(rows, keys)
    store[f"{name}/nfeat"] = np.array([len(keys)])
    for f, (v, o) in enumerate(feats):
        store[f"{name}/in{f}_values"] = v
        store[f"{name}/in{f}_offsets"] = o
        jt = ik.per_feature[keys[f]]
        store[f"{name}/out{f}_values"] = np.array(jt.values)
        store[f"{name}/out{f}_offsets"] = np.array(jt.offsets)
    store[f"{name}/inverse"] = np.array(ik.inverse_lookup)


def session_rows(rng, b, keys, dup_rate, max_len, vocab, long_every=0):
    rows, state = [], None
    for i in range(b):
        if state is None or rng.random() > dup_rate:
            state = {}
            for k in keys:
                n = int(rng.integers(0, max_len + 1))
                if long_every and rng.random() < 1.0 / long_every:
                    n = int(rng.integers(100, 300))
                state[k] = rng.integers(0, vocab, size=n).tolist()
        rows.append(dict(state))
    return rows


def make_dedup():
    store = {}
    rows = [
        {"a": [1, 2], "b": [3, 4, 5], "c": [7, 8], "d": [9]},
        {"a": [], "b": [4, 5, 6], "c": [7, 8], "d": [9]},
        {"a": [1, 2], "b": [3, 4, 5], "c": [10], "d": [11]},
    ]  # test_tensors.py:32-36 (paper Fig. 5)
    names = []
    for keys in (["b"], ["c", "d"], ["a"], ["a", "b", "c", "d"]):
        nm = "worked_" + "".join(keys)
        _store_case(store, nm, keys, rows)
        names.append(nm)
    extra = {
        "first_occ": ([{"a": [5]}, {"a": [3]}, {"a": [5]}, {"a": [1]}, {"a": [3]}], ["a"]),
        "len_boundary": ([{"x": [1, 2], "y": [3]}, {"x": [1], "y": [2, 3]}], ["x", "y"]),
        "unsync": ([{"c": [7, 8], "e": [1]}, {"c": [7, 8], "e": [2]}], ["c", "e"]),
        "distinct": ([{"a": [i]} for i in range(5)], ["a"]),
        "empties": ([{"a": []}, {}, {"a": [1]}, {"a": []}, {"a": [1]}, {}], ["a"]),
        "single": ([{"x": [7]}], ["x"]),
        "all_empty": ([{} for _ in range(7)], ["p", "q"]),
    }
    for nm, (rws, keys) in extra.items():
        _store_case(store, nm, keys, rws)
        names.append(nm)
    rng = np.random.default_rng(20261018)
    for c in range(48):
        b = int(rng.choice([1, 2, 3, 31, 32, 33, 100, 257, 1000, 2048, 4096]))
        width = int(rng.integers(1, 4))
        keys = [f"f{j}" for j in range(width)]
        vocab = int(rng.choice([3, 6, 50, 1_000_000]))
        max_len = int(rng.choice([0, 1, 4, 8, 40]))
        rws = session_rows(rng, b, keys, float(rng.uniform(0.2, 0.95)), max_len, vocab,
                           long_every=int(rng.choice([0, 0, 50])))
        nm = f"rand{c}"
        _store_case(store, nm, keys, rws)
        names.append(nm)
    store["names"] = np.array(names)
    np.savez_compressed(OUT / "dedup.npz", **store)


def make_datagen():
    """cfg1 inputs via the reference generator, clustered."""
    store = {}
    for tag, specs, nsess, b, dist in (
        ("cfg1", [DG.FeatureSpec(f"k{i}", "user_sequence", float(L), 1_000_000, 0.15)
                  for i, L in enumerate([4, 8, 12, 16, 20, 24, 28, 32])], 600, 4096,
         DG.SampleCountDist("geometric", 16.5)),
        ("mixed", [DG.FeatureSpec("u", "user_sequence", 3.5, 50, 0.3, sync_group="g"),
                   DG.FeatureSpec("v", "user_sequence", 2.0, 50, 0.3, sync_group="g"),
                   DG.FeatureSpec("w", "user_sequence", 5.0, 1000, 0.5),
                   DG.FeatureSpec("it", "item", 2.5, 100)], 80, 500,
         DG.SampleCountDist("fixed", 8)),
    ):
        cfg = DG.SessionConfig(num_sessions=nsess, samples_per_session=dist, seed=0)
        recs = DG.generate_dataset(cfg, specs)
        recs.sort(key=lambda r: (r.session_id, r.timestamp))
        rows = recs[:b]
        keys = [s.key for s in specs]
        kjt = T.build_kjt(rows, keys)
        for k in keys:
            v = np.array(kjt.entries[k].values)
            o = np.array(kjt.entries[k].offsets)
            store[f"{tag}/{k}/sha"] = np.array(
                [hashlib.sha256(v.tobytes() + o.tobytes()).hexdigest()])
        store[f"{tag}/session_ids"] = np.array([r.session_id for r in rows])
        store[f"{tag}/labels"] = np.array([r.label for r in rows])
        if tag == "cfg1":
            for k in keys:
                ik = T.build_ikjt(rows, [k])
                jt = ik.per_feature[k]
                store[f"{tag}/{k}/inverse"] = np.array(ik.inverse_lookup).astype(np.int32)
                store[f"{tag}/{k}/uoffsets"] = np.array(jt.offsets).astype(np.int32)
                store[f"{tag}/{k}/uvalues"] = np.array(jt.values).astype(np.int32)
    # reference-seeded table init (trainer_sim.py:62-66, 83-87)
    t = TS.EmbeddingTable.create("k0", rows=64, dim=8, seed=0)
    store["table_k0_64x8"] = np.array(t.weights)
    np.savez_compressed(OUT / "datagen.npz", **store)


def make_pool():
    store = {}
    rng = np.random.default_rng(7)
    lens_all = (list(range(0, 21)) + list(range(127, 138)) + list(range(255, 265))
                + [300, 513])
    for dim in (1, 4, 8, 64, 128):
        rows = 512
        table = TS.EmbeddingTable.create(f"t{dim}", rows=rows, dim=dim, seed=3)
        lens = np.array(lens_all + list(rng.integers(0, 40, size=24)), dtype=np.int64)
        rng.shuffle(lens)
        vals = rng.integers(0, rows, size=int(lens.sum())).astype(np.int64)
        offs = np.zeros(lens.size, dtype=np.int64)
        np.cumsum(lens[:-1], out=offs[1:])
        jt = T.JaggedTensor(values=vals, offsets=offs)
        acts = TS.embedding_lookup(jt, table, f"t{dim}")
        store[f"d{dim}/weights"] = np.array(table.weights)
        store[f"d{dim}/values"] = vals
        store[f"d{dim}/offsets"] = offs
        inv = rng.integers(0, lens.size, size=3 * lens.size).astype(np.int64)
        inv[: lens.size] = np.arange(lens.size)
        rng.shuffle(inv)
        store[f"d{dim}/inverse"] = inv
        for op in ("sum", "avg", "max"):
            pooled = TS.pool(acts, jt.offsets, op)
            store[f"d{dim}/{op}"] = pooled
            store[f"d{dim}/{op}_expanded"] = pooled[inv]
    np.savez_compressed(OUT / "pool.npz", **store)


def make_jagged():
    store = {}
    rng = np.random.default_rng(5)
    n = 0
    for _ in range(300):
        n_rows = int(rng.integers(1, 12))
        rows = [rng.integers(0, 50, size=rng.integers(0, 6)).tolist() for _ in range(n_rows)]
        jt = T.JaggedTensor.from_rows(rows)
        idx = rng.integers(0, n_rows, size=rng.integers(0, 20)).astype(np.int64)
        out = T.jagged_index_select(jt, idx)
        for nm, arr in (("values", jt.values), ("offsets", jt.offsets), ("idx", idx),
                        ("out_values", out.values), ("out_offsets", out.offsets)):
            store[f"c{n}/{nm}"] = np.array(arr, dtype=np.int64)
        n += 1
    store["count"] = np.array([n])
    np.savez_compressed(OUT / "jagged.npz", **store)


def make_slice():
    store = {}
    rng = np.random.default_rng(11)
    cases = []
    for c in range(30):
        b = int(rng.integers(2, 300))
        rws = session_rows(rng, b, ["u", "v"], 0.7, 4, 20)
        ik = T.build_ikjt(rws, ["u", "v"])
        a = int(rng.integers(0, b - 1))
        z = int(rng.integers(a + 1, b + 1))
        sub = TS.slice_ikjt_rows(ik, a, z)
        store[f"c{c}/inverse"] = np.array(ik.inverse_lookup)
        for f, k in enumerate(["u", "v"]):
            store[f"c{c}/in{f}_values"] = np.array(ik.per_feature[k].values)
            store[f"c{c}/in{f}_offsets"] = np.array(ik.per_feature[k].offsets)
            store[f"c{c}/out{f}_values"] = np.array(sub.per_feature[k].values)
            store[f"c{c}/out{f}_offsets"] = np.array(sub.per_feature[k].offsets)
        store[f"c{c}/range"] = np.array([a, z])
        store[f"c{c}/out_inverse"] = np.array(sub.inverse_lookup)
        cases.append(c)
    store["count"] = np.array([len(cases)])
    np.savez_compressed(OUT / "slice.npz", **store)


def make_errors():
    msgs = {}

    def cap(name, fn):
        try:
            fn()
        except Exception as e:  # noqa: BLE001
            msgs[name] = [type(e).__name__, str(e)]

    cap("empty_batch", lambda: T.build_ikjt([], ["a"]))
    cap("empty_group", lambda: T.build_ikjt([{"a": [1]}], []))
    cap("kjt_empty_batch", lambda: T.build_kjt([], ["a"]))
    cap("index_oob", lambda: T.jagged_index_select(
        T.JaggedTensor.from_rows([[1], [2]]), np.array([0, 5, -1])))
    tbl = TS.EmbeddingTable(key="b", rows=4, dim=1,
                            weights=np.arange(4, dtype=np.float32).reshape(-1, 1))
    cap("id_oob", lambda: TS.embedding_lookup(T.JaggedTensor.from_rows([[1], [9], [3]]), tbl, "b"))
    cap("pool_op", lambda: TS.pool(np.zeros((1, 1), dtype=np.float32), np.array([0]), "median"))
    cap("slice_range", lambda: TS.slice_ikjt_rows(T.build_ikjt([{"f": [1]}], ["f"]), 0, 2))
    np.savez_compressed(OUT / "errors.npz", json=np.array([json.dumps(msgs)]))


def make_transforms():
    """reader.apply_transform (reader.py:69-81) on edge and random int64 IDs,
    and reader.process on an IKJT: transformed dedup values, expanded, equal
    the transformed KJT (test_reader.py:176-187)."""
    rng = np.random.default_rng(11)
    v = np.concatenate([
        np.array([0, 1, -1, 2**63 - 1, -2**63, 12345678901234, 10_000_000, 9_999_999], np.int64),
        rng.integers(-2**63, 2**63 - 1, size=2000, dtype=np.int64),
        rng.integers(0, 10_000_000, size=2000, dtype=np.int64)])
    store = {"values": v}
    cases = [("identity", None), ("mod_hash", 1), ("mod_hash", 1000), ("mod_hash", 10_000_000),
             ("mod_hash", 2**62 + 7), ("clamp", 1), ("clamp", 5_000_000), ("clamp", 2**62)]
    for i, (op, param) in enumerate(cases):
        t = RD.Transform(op=op, key="k", param=param)
        store[f"c{i}/op"] = np.array([op])
        store[f"c{i}/param"] = np.array([param if param is not None else 0], np.int64)
        store[f"c{i}/out"] = np.asarray(RD.apply_transform(v, t), dtype=np.int64)
    store["ncases"] = np.array([len(cases)])
    np.savez_compressed(OUT / "transforms.npz", **store)


def make_wire():
    """Canonical wire format (tensors.py:463-515) of KJTs and IKJTs built by the
    real reference: serialize_kjt / serialize_ikjt bytes + slice byte counts."""
    rng = np.random.default_rng(13)
    store = {}
    cases = []
    for ci, (b, keys, dup) in enumerate([(1, ["a"], 0.0), (7, ["user_hist", "x"], 0.7),
                                         (300, ["k0", "k1", "k_\u00e9"], 0.85), (64, ["e"], 0.5)]):
        rows = session_rows(rng, b, keys, dup, 12, 1 << 40)
        if ci == 3:  # rows with only empty lists
            rows = [{"e": []} for _ in range(b)]
        kjt = T.build_kjt(rows, keys)
        ik = T.build_ikjt(rows, keys)
        name = f"w{ci}"
        store[f"{name}/kjt_bytes"] = np.frombuffer(T.serialize_kjt(kjt), np.uint8)
        store[f"{name}/ikjt_bytes"] = np.frombuffer(T.serialize_ikjt(ik), np.uint8)
        store[f"{name}/keys"] = np.array(keys)
        store[f"{name}/slice_bytes"] = np.array([T.slice_stream_bytes(ik.per_feature[k]) for k in keys], np.int64)
        store[f"{name}/values_bytes"] = np.array([T.values_stream_bytes(ik.per_feature[k]) for k in keys],
                                                 np.int64)
        for k in keys:
            store[f"{name}/in_{k}_values"] = kjt.entries[k].values
            store[f"{name}/in_{k}_offsets"] = kjt.entries[k].offsets
        cases.append(name)
    store["names"] = np.array(cases)
    np.savez_compressed(OUT / "wire.npz", **store)


def make_sdd():
    """IterationStats of the real forward_iteration (trainer_sim.py:484-586):
    the sdd all-to-all bytes (trainer_sim.py:281-305), the pooled rows sent
    back, lookups, activation peak, pooling MACs and index-select elements,
    dedup vs baseline, R in {1, 2, 4, 8} ranks, element + attention pooling +
    a plain key.  Inputs: the reference generator's clustered records."""
    specs = [DG.FeatureSpec("u", "user_sequence", 3.5, 60, 0.3, sync_group="g"),
             DG.FeatureSpec("v", "user_sequence", 2.0, 60, 0.3, sync_group="g"),
             DG.FeatureSpec("w", "user_sequence", 6.5, 3000, 0.25),
             DG.FeatureSpec("x", "user_sequence", 12.0, 3000, 0.1),
             DG.FeatureSpec("y", "user_sequence", 4.0, 3000, 0.4),
             DG.FeatureSpec("it", "item", 2.5, 500)]
    cfg = DG.SessionConfig(num_sessions=90, samples_per_session=DG.SampleCountDist("geometric", 8.0),
                           seed=3)
    recs = DG.generate_dataset(cfg, specs)
    recs.sort(key=lambda r: (r.session_id, r.timestamp))
    rows = recs[:403]          # not a multiple of 8: split_batch's uneven chunks
    keys = [s.key for s in specs]
    dim = 8
    spec = TS.ModelSpec(
        tables={k: TS.TableConfig(rows=s.vocab_size, dim=dim) for k, s in zip(keys, specs)},
        groups=(TS.GroupConfig(("u", "v"), "attention"), TS.GroupConfig(("w",), "sum"),
                TS.GroupConfig(("x",), "avg"), TS.GroupConfig(("y",), "max")),
        plain={"it": "sum"}, seed=0)
    rspec = RD.DataloaderSpec(keys=tuple(keys),
                              dedup_sparse_features=(("u", "v"), ("w",), ("x",), ("y",)),
                              batch_size=len(rows))
    store = {"rows/keys": np.array(keys), "dim": np.array([dim])}
    kjt = T.build_kjt(rows, keys)
    for k in keys:
        store[f"in/{k}/values"] = np.array(kjt.entries[k].values)
        store[f"in/{k}/offsets"] = np.array(kjt.entries[k].offsets)
    fields = ["a2a_bytes_fwd", "a2a_bytes_back", "lookup_count", "activation_elements",
              "pooling_mac_count", "index_select_elements"]
    store["fields"] = np.array(fields)
    tables = TS.build_tables(spec)
    for mode, rs in (("dedup", rspec), ("baseline", rspec.without_dedup())):
        batch = RD.convert(rows, rs)
        for R in (1, 2, 4, 8):
            plan = TS.make_round_robin_plan(spec, R)
            scores, st = TS.forward_iteration(batch, spec, plan, mode, tables)
            store[f"{mode}/R{R}/stats"] = np.array([getattr(st, f) for f in fields], dtype=np.int64)
            store[f"{mode}/R{R}/plan"] = np.array([plan.assignment[k] for k in keys])
            store[f"{mode}/R{R}/scores"] = scores
    np.savez_compressed(OUT / "sdd.npz", **store)


def shifted_sessions(rng, b, vocab, max_len, p_shift=(0.5, 0.35, 0.15), mean_session=8.0):
    """Session-structured rows of one key: each session draws a length and a
    value pool; consecutive rows shift the window by 0, 1 or 2 (the reference
    datagen's shift model, datagen.py:149-183, with 2-shifts added)."""
    rows = []
    while len(rows) < b:
        n = int(rng.integers(0, max_len + 1))
        count = 1 + int(rng.poisson(mean_session - 1))
        shifts = np.concatenate([[0], np.cumsum(rng.choice(3, size=count - 1, p=p_shift))]).astype(np.int64)
        pool = rng.integers(-vocab // 4, vocab, size=n + int(shifts[-1]))
        for s in shifts[: b - len(rows)]:
            rows.append({"f": pool[s:s + n].tolist()})
    return rows


def make_partial():
    """Partial IKJT (tensors.py:311-360) of the real reference: values + windows."""
    rng = np.random.default_rng(17)
    cases = {
        "p0": [[3, 4, 5], [4, 5, 6], [3, 4, 5]],
        "p1": [[3, 4, 5], [4, 5, 6], [1], []],
        "p2": [[9, 9], [9, 9]],
        "p4": [[1, 2, 3, 4, 5], [2, 3], [3, 4, 5], [5], [4, 5, 6], [1, 2], [6, 7], [], [7], [5, 6, 7, 8]],
        "p5": [[1], [2], [1, 2, 3], [3], [2, 3, 4, 5], [9], [3, 4, 5, 9, 1], [4, 5, 9, 1, 7], [1, 7]],
        "p6": [[]] * 5,
        "p9": [[-(2 ** 63), 2 ** 63 - 1], [2 ** 63 - 1, 0], [0, -(2 ** 63)], [-(2 ** 63), 2 ** 63 - 1, 0]],
    }
    pool = rng.integers(0, 10_000, size=400, dtype=np.int64)
    rows, start = [], 0
    for _ in range(40):
        start += int(rng.integers(0, 3))
        rows.append(pool[start:start + 20].tolist())
    cases["p3"] = rows
    cases["p7"] = [rng.integers(-1, 3, size=int(rng.integers(0, 7))).tolist() for _ in range(300)]
    cases["p8"] = [r["f"] for r in shifted_sessions(rng, 400, 50, 12)]
    cases["p10"] = [r["f"] for r in shifted_sessions(rng, 2000, 1 << 40, 64)]
    cases["p11"] = [r["f"] for r in shifted_sessions(rng, 1500, 6, 9, p_shift=(0.2, 0.5, 0.3), mean_session=4.0)]
    store = {}
    for name, lists in cases.items():
        recs = [{"f": x} for x in lists]
        kjt = T.build_kjt(recs, ["f"])
        pk = T.build_partial_ikjt(recs, "f")
        store[f"{name}/in_values"] = np.array(kjt.entries["f"].values)
        store[f"{name}/in_offsets"] = np.array(kjt.entries["f"].offsets)
        store[f"{name}/values"] = np.array(pk.values)
        store[f"{name}/windows"] = np.array(pk.windows)
    store["names"] = np.array(list(cases))
    np.savez_compressed(OUT / "partial.npz", **store)


if __name__ == "__main__":
    makers = {"partial": make_partial, "wire": make_wire, "transforms": make_transforms,
              "dedup": make_dedup, "datagen": make_datagen, "pool": make_pool,
              "jagged": make_jagged, "slice": make_slice, "errors": make_errors, "sdd": make_sdd}
    for name in (sys.argv[1:] or list(makers)):   # e.g. `make_golden.py sdd`
        makers[name]()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
