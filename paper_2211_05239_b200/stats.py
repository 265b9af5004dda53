"""Per-iteration exchange and work counters of the sparse path.

Drop-in for the reference's `IterationStats`, `make_round_robin_plan`,
`split_batch` chunking and the byte accounting of `sdd` / `forward_iteration`
(/root/reference/pkg/src/sessiondedup/trainer_sim.py:202-242, 281-305,
416-446, 484-586): the reference computes them while it moves numpy slices;
here they are computed from the device-resident sizes of the IKJTs the
kernels produced (unique rows U and unique values N_u per chunk and key, and
for attention groups the per-unique-row sequence lengths, reduced on the
GPU), so a step never has to materialise the exchanged tensors on the host.

Counters (per iteration, all source ranks):
  a2a_bytes_fwd          sum over keys and sources of the canonical wire size
                         of the transmitted (offsets, values) slice,
                         16 + 8 (rows + values) (tensors.py:507-510); local
                         destinations included, the inverse never travels
  a2a_bytes_back         pooled rows returned: rows x dim x 4 per block
  lookup_count           embedding rows gathered (values of every slice)
  activation_elements    peak values x dim of one (source, key) slice
  pooling_mac_count      values x dim per element-pooled slice; attention:
                         3 n d^2 + 2 n^2 d + d^2 per non-empty unique row
  index_select_elements  B_src x dim per pooled block of a group (the
                         inverse expansion; plain keys have none)
"""

from __future__ import annotations

from dataclasses import dataclass, fields
from typing import Mapping, Sequence

__all__ = ["IterationStats", "round_robin_plan", "split_bounds", "iteration_stats",
           "chunk_sizes", "attention_macs", "ikjt_attention_macs", "STAT_FIELDS"]


@dataclass
class IterationStats:
    """trainer_sim.py:217-234."""

    a2a_bytes_fwd: int = 0
    a2a_bytes_back: int = 0
    lookup_count: int = 0
    activation_elements: int = 0
    pooling_mac_count: int = 0
    index_select_elements: int = 0

    def dominated_by(self, other: "IterationStats") -> bool:
        """True when every counter here is <= the other's."""
        return all(getattr(self, f.name) <= getattr(other, f.name) for f in fields(self))

    def as_list(self) -> list[int]:
        return [int(getattr(self, f.name)) for f in fields(self)]


STAT_FIELDS = tuple(f.name for f in fields(IterationStats))


def round_robin_plan(groups: Sequence[Sequence[str]], plain: Sequence[str],
                     num_ranks: int) -> dict[str, int]:
    """make_round_robin_plan (trainer_sim.py:202-214): groups, then plain
    keys, dealt round-robin; a group's keys share one rank."""
    if num_ranks < 1:
        raise ValueError("num_ranks must be >= 1")
    out: dict[str, int] = {}
    unit = 0
    for g in groups:
        for k in g:
            out[k] = unit % num_ranks
        unit += 1
    for k in plain:
        out[k] = unit % num_ranks
        unit += 1
    return out


def split_bounds(batch_size: int, num_ranks: int) -> list[tuple[int, int]]:
    """split_batch's contiguous chunks (trainer_sim.py:416-446): the first
    B mod R chunks take one extra row."""
    if num_ranks < 1:
        raise ValueError("num_ranks must be >= 1")
    if batch_size < num_ranks:
        raise ValueError(f"cannot split {batch_size} rows across {num_ranks} ranks")
    base, extra = divmod(batch_size, num_ranks)
    out, start = [], 0
    for r in range(num_ranks):
        stop = start + base + (1 if r < extra else 0)
        out.append((start, stop))
        start = stop
    return out


def chunk_sizes(ikjts, kjt=None) -> dict[str, tuple[int, int]]:
    """(rows, values) of every transmitted slice of one source chunk: the
    unique rows / values of each IKJT feature, the rows / values of each
    plain KJT key (all host-known sizes of device tensors)."""
    out = {}
    for ik in ikjts:
        for k in ik.group_keys:
            jt = ik.per_feature[k]
            out[k] = (int(jt.row_count), int(jt.values.numel()))
    if kjt is not None:
        for k, jt in kjt.entries.items():
            out[k] = (int(jt.row_count), int(jt.values.numel()))
    return out


def attention_macs(lengths, dim: int) -> int:
    """sum over the unique rows of an attention group of 3 n d^2 + 2 n^2 d +
    d^2, n = the row's concatenated sequence length (trainer_sim.py:386-390).
    `lengths`: per group feature, the unique rows' lengths -- torch tensors
    (IKJT.per_feature[k].row_lengths(), reduced on the device) or numpy."""
    n = None
    for ln in lengths:
        n = ln if n is None else n + ln
    d = int(dim)
    nz = n[n > 0]
    return int((3 * nz * d * d + 2 * nz * nz * d + d * d).sum())


def ikjt_attention_macs(ikjt, dim: int) -> int:
    """attention_macs of a device IKJT (one host read of the sum)."""
    return attention_macs([ikjt.per_feature[k].row_lengths() for k in ikjt.group_keys], dim)


def iteration_stats(groups: Sequence[tuple[Sequence[str], str]], plain: Mapping[str, str],
                    dim: int, sizes: Sequence[Mapping[str, tuple[int, int]]],
                    batch_sizes: Sequence[int],
                    attention_mac: Mapping[tuple[int, int], int] | None = None) -> IterationStats:
    """IterationStats of one forward_iteration (trainer_sim.py:484-586).

    groups        [(keys, pooling)] in model order; pooling "attention" or element-wise
    plain         {key: pooling} of the keys sent as plain KJT rows
    sizes[r]      {key: (rows, values)} of source chunk r's transmitted slice
                  (dedup: unique rows / values; baseline: batch rows / values)
    batch_sizes   B_r of every chunk
    attention_mac {(r, group index): MACs} of attention groups (attention_macs)
    """
    st = IterationStats()
    d = int(dim)
    R = len(sizes)
    for r in range(R):
        for k, (rows, vals) in sizes[r].items():
            st.a2a_bytes_fwd += 16 + 8 * (rows + vals)
    for gi, (keys, pooling) in enumerate(groups):
        for r in range(R):
            for k in keys:
                rows, vals = sizes[r][k]
                st.lookup_count += vals
                st.activation_elements = max(st.activation_elements, vals * d)
            urows = sizes[r][keys[0]][0]
            if pooling == "attention":
                st.pooling_mac_count += int((attention_mac or {})[(r, gi)])
                nblocks = 1
            else:
                for k in keys:
                    st.pooling_mac_count += sizes[r][k][1] * d
                nblocks = len(keys)
            st.a2a_bytes_back += nblocks * urows * d * 4
            st.index_select_elements += nblocks * int(batch_sizes[r]) * d
    for k in plain:
        for r in range(R):
            rows, vals = sizes[r][k]
            st.lookup_count += vals
            st.activation_elements = max(st.activation_elements, vals * d)
            st.pooling_mac_count += vals * d
            st.a2a_bytes_back += rows * d * 4
    return st
