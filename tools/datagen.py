"""Synthetic session-structured KJT batches (input generator, not product path).

Restates the reference generator (`/root/reference/pkg/src/sessiondedup/
datagen.py`) so that the GPU box -- where `/root/reference` does not exist --
can build the same inputs: every session owns a child RNG
``default_rng(SeedSequence((seed, idx)))`` (datagen.py:206-207) and draws, in
order, its sample count (99-104), timestamps over a shared horizon (258-260),
labels (261), one mutation-coin sequence per sync group (223-228), then per
feature either a shift-append window pool (user_sequence, 229-239) or fresh
per-impression lists (item, 240-249).  The RNG call sequence is identical, so
for the same (config, num_sessions) the feature lists are bit-identical to the
reference's (pinned by `tests/test_datagen.py` against a checksum recorded
from the real reference in `tests/golden/`).

Instead of materialising one ``ImpressionRecord`` per row, batches are emitted
directly in KJT form (int64 values + one offset per row) in session-clustered
order, i.e. the reference's records sorted by ``(session_id, timestamp)``
(SURVEY.md §8(d) "cfg1 inputs").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "FeatureSpec",
    "SampleCountDist",
    "SessionConfig",
    "ClusteredBatch",
    "generate_clustered_batch",
    "cfg1_specs",
    "cfg2_specs",
]

_LABEL_RATE = 0.1  # datagen.py:38


@dataclass(frozen=True)
class FeatureSpec:
    """datagen.py:41-76 (validation kept minimal; kinds as in the reference)."""

    key: str
    kind: str  # "user_sequence" | "item"
    avg_len: float
    vocab_size: int
    change_prob: float = 0.0
    sync_group: str | None = None


@dataclass(frozen=True)
class SampleCountDist:
    """datagen.py:79-117 ("fixed" | "geometric")."""

    kind: str
    mean: float = 1.0

    def sample(self, rng: np.random.Generator) -> int:
        if self.kind == "fixed":
            return int(self.mean)
        if self.kind == "geometric":
            return int(rng.geometric(1.0 / self.mean))
        raise ValueError(f"unsupported distribution kind {self.kind!r}")


@dataclass(frozen=True)
class SessionConfig:
    num_sessions: int
    samples_per_session: SampleCountDist
    seed: int = 0


@dataclass
class ClusteredBatch:
    """One session-clustered batch in KJT layout (numpy, host)."""

    batch_size: int
    keys: tuple[str, ...]
    values: dict[str, np.ndarray]   # int64[N_k]
    offsets: dict[str, np.ndarray]  # int64[B]
    session_ids: np.ndarray         # int64[B]
    labels: np.ndarray              # int64[B]


def _draw_length(avg_len: float, rng: np.random.Generator) -> int:
    """datagen.py:196-200."""
    base = int(avg_len)
    frac = avg_len - base
    return base + (1 if frac > 0 and rng.random() < frac else 0)


def _session_rng(seed: int, index: int) -> np.random.Generator:
    """datagen.py:206-207."""
    return np.random.default_rng(np.random.SeedSequence((seed, index)))


def _gen_session(count: int, specs, rng):
    """datagen.py:210-250, emitting per-feature (values, lengths) blocks."""
    group_of = {
        s.key: (s.sync_group if s.sync_group is not None else f"_solo_{s.key}")
        for s in specs if s.kind == "user_sequence"
    }
    coins: dict[str, np.ndarray] = {}
    for s in specs:
        if s.kind != "user_sequence":
            continue
        g = group_of[s.key]
        if g not in coins:
            coins[g] = rng.random(count - 1) < s.change_prob
    out = {}
    for s in specs:
        if s.kind == "user_sequence":
            length = _draw_length(s.avg_len, rng)
            flips = coins[group_of[s.key]]
            shifts = np.zeros(count, dtype=np.int64)
            if count > 1:
                np.cumsum(flips, out=shifts[1:])
            pool = rng.integers(0, s.vocab_size, length + int(shifts[-1]), dtype=np.int64)
            idx = shifts[:, None] + np.arange(length, dtype=np.int64)[None, :]
            out[s.key] = (pool[idx].reshape(-1), np.full(count, length, dtype=np.int64))
        else:
            lengths = np.array([_draw_length(s.avg_len, rng) for _ in range(count)], dtype=np.int64)
            flat = rng.integers(0, s.vocab_size, int(lengths.sum()), dtype=np.int64)
            out[s.key] = (flat, lengths)
    return out


def generate_clustered_batch(cfg: SessionConfig, specs, batch_size: int,
                             row_start: int = 0) -> ClusteredBatch:
    """Rows ``[row_start, row_start + batch_size)`` of the session-clustered
    record stream of ``generate_dataset(cfg, specs)`` (datagen.py:253-283,
    re-sorted by (session_id, timestamp)).  ``row_start`` lets DP rank r take
    its contiguous chunk, as `split_batch` does (trainer_sim.py:416-446)."""
    keys = tuple(s.key for s in specs)
    mean_s = cfg.samples_per_session.mean
    horizon = max(64, int(4 * cfg.num_sessions * mean_s))  # datagen.py:257
    row_stop = row_start + batch_size
    vals = {k: [] for k in keys}
    lens = {k: [] for k in keys}
    sids, labs = [], []
    pos = 0
    for idx in range(cfg.num_sessions):
        if pos >= row_stop:
            break
        rng = _session_rng(cfg.seed, idx)
        count = cfg.samples_per_session.sample(rng)
        if pos + count <= row_start:
            pos += count
            continue
        rng.integers(0, horizon, count)  # timestamps: consumed, not needed
        labels = rng.random(count) < _LABEL_RATE
        feats = _gen_session(count, specs, rng)
        lo = max(0, row_start - pos)
        hi = min(count, row_stop - pos)
        for k in keys:
            v, ln = feats[k]
            bounds = np.zeros(count + 1, dtype=np.int64)
            np.cumsum(ln, out=bounds[1:])
            vals[k].append(v[bounds[lo]:bounds[hi]])
            lens[k].append(ln[lo:hi])
        sids.append(np.full(hi - lo, idx, dtype=np.int64))
        labs.append(labels[lo:hi].astype(np.int64))
        pos += count
    if pos < row_stop:
        raise ValueError(f"{cfg.num_sessions} sessions give only {pos} rows (< {row_stop})")
    values, offsets = {}, {}
    for k in keys:
        ln = np.concatenate(lens[k])
        off = np.zeros(batch_size, dtype=np.int64)
        if batch_size > 1:
            np.cumsum(ln[:-1], out=off[1:])
        values[k] = np.ascontiguousarray(np.concatenate(vals[k]), dtype=np.int64)
        offsets[k] = off
    return ClusteredBatch(batch_size, keys, values, offsets,
                          np.concatenate(sids), np.concatenate(labs))


def cfg1_specs() -> list[FeatureSpec]:
    """BASELINE.json configs[0] / SURVEY.md §8(d) cfg1: 8 keys, L=4..32, vocab 1M."""
    return [FeatureSpec(f"k{i}", "user_sequence", float(L), 1_000_000, 0.15)
            for i, L in enumerate([4, 8, 12, 16, 20, 24, 28, 32])]


def cfg2_specs(vocab: int = 10_000_000, change_prob: float = 0.15) -> list[FeatureSpec]:
    """BASELINE.json configs[1] / SURVEY.md §8(d) cfg2: 26 keys, L up to 256."""
    lens = ([8, 16, 32, 64, 128, 256] * 5)[:26]
    return [FeatureSpec(f"k{i}", "user_sequence", float(L), vocab, change_prob)
            for i, L in enumerate(lens)]
