// KJT -> IKJT deduplication on sm_100a (replaces tensors.build_ikjt,
// /root/reference/pkg/src/sessiondedup/tensors.py:269-308).
//
// Semantics kept exactly: rows i, j of a group merge iff every feature list
// (length included, `_pack_group_row` tensors.py:257-262) is equal; unique
// rows are numbered in first-occurrence order (tensors.py:289-298); a hash
// never merges unequal rows (full compare on hash match, tensors.py:270-276).
//
// Pipeline (one launch per phase for all groups of the step):
//   k_rowscan  (group, 256-row chunk) blocks stream the KJT values once
//              (8 consecutive values per thread, 128-bit loads) and compare
//              each row with its predecessor: head[i] = row i differs from row
//              i-1 (session-clustered batches make ~80% of rows non-heads); the
//              block also clears its slice of the group's hash table.
//              A second pass hashes the chunk's heads (warp per head row).
//   k_insert   heads only: open-addressing table (64-bit key, L2 resident),
//              rep = atomicMin(row) per key.
//   k_resolve  heads whose rep != self are fully compared with the rep; a
//              mismatch (a true 64-bit collision) is marked pending.
//   k_fallback (cold) exact sequential resolution of pending heads.
//   k_num_*    chunk-parallel numbering: run-head propagation, first-occurrence
//              uids, unique offsets per feature, inverse (reduce/scan/down).
//   k_copy     value-parallel gather of the unique lists into the unique values.
#include <algorithm>
#include <vector>

#include "recd_common.cuh"

namespace recd {

uint64_t g_hash_mask = ~0ull;

struct DedupParams {
  int G, F;
  int64_t B;
  int64_t C;  // hash-table slots per group (power of two >= 2B)
  uint64_t hash_mask;
  int group_first[RECD_MAX_FEAT + 1];
  int feat_group[RECD_MAX_FEAT];
  const int64_t* values[RECD_MAX_FEAT];
  const int64_t* offsets[RECD_MAX_FEAT];
  int64_t nvalues[RECD_MAX_FEAT];  // host: value counts, or capacities when nv_dev is set
  const int64_t* nv_dev;            // device [F] value counts (one graph for any batch), or null
  int64_t* inverse[RECD_MAX_FEAT];
  int64_t* uoffsets[RECD_MAX_FEAT];
  int64_t* uvalues[RECD_MAX_FEAT];
  int64_t* count_rows;  // [F] U per feature
  int64_t* count_vals;  // [F] N_u per feature
  uint8_t* head;        // [G][B]
  uint64_t* hash;       // [G][B]
  uint32_t* slot_of;    // [G][B]
  int32_t* cls;         // [G][B]  class representative (min row of the class)
  int32_t* uidmap;      // [G][B]
  int32_t* first_rows;  // [G][B]
  int64_t* nb_rh;       // [G][nch] numbering chunk aggregates
  int64_t* nb_nf;       // [G][nch]
  int64_t* nb_len;      // [F][nch]
  int nb_ch;            // rows per numbering chunk (NB_NT * items)
  int32_t* fb_list;     // [G][B]
  unsigned long long* tkeys;  // [G][C]
  uint32_t* treps;            // [G][C]
  int32_t* collide;           // [G]
  int rs_group[RECD_MAX_FEAT];
  int64_t cp_blk0[RECD_MAX_FEAT + 1];  // k_copy: first block of each feature
  int64_t cp_ch;                       // k_copy: unique values per block
  // k_copy second destination (fused shard dispatch): values also go to
  // rdst[f][*rbase[f] + j] (peer memory of the feature's owner), or null
  int64_t* rdst[RECD_MAX_FEAT];
  const int64_t* rbase[RECD_MAX_FEAT];  // k_rowscan: groups in launch order (most values first)
};

// number of KJT values of feature f (the last row runs to it, tensors.py:65-66)
__device__ __forceinline__ int64_t nval(const DedupParams& p, int f) {
  return p.nv_dev ? __ldg(p.nv_dev + f) : p.nvalues[f];
}

__device__ __forceinline__ int64_t row_begin(const int64_t* off, int64_t i) { return off[i]; }
__device__ __forceinline__ int64_t row_end(const int64_t* off, int64_t i, int64_t B, int64_t nv) {
  return (i + 1 < B) ? off[i + 1] : nv;
}

__device__ bool rows_equal(const DedupParams& p, int g, int64_t a, int64_t b) {
  for (int f = p.group_first[g]; f < p.group_first[g + 1]; ++f) {
    const int64_t* off = p.offsets[f];
    const int64_t* val = p.values[f];
    int64_t sa = off[a], ea = row_end(off, a, p.B, nval(p, f));
    int64_t sb = off[b], eb = row_end(off, b, p.B, nval(p, f));
    if (ea - sa != eb - sb) return false;
    for (int64_t k = 0; k < ea - sa; ++k)
      if (val[sa + k] != val[sb + k]) return false;
  }
  return true;
}

__device__ __forceinline__ uint64_t finalize_hash(uint64_t h, uint64_t mask) {
  uint64_t x = mix64(h) & mask;
  return x ? x : 1ull;  // 0 marks an empty table slot
}

// ---------------------------------------------------------------- rowscan
// Compare-only pass over the KJT values: block per (group, 256-row chunk),
// 8 consecutive values per thread (128-bit loads), each compared with the
// same position of the previous row (q - len; an L1 hit for rows shorter
// than a tile).  Only run heads need a content hash, and they are ~20% of the
// rows of a session-clustered batch, so hashing is deferred to k_insert.
#ifndef RECD_RS_RPB
#define RECD_RS_RPB 256
#endif
#ifndef RECD_RS_IT
#define RECD_RS_IT 8
#endif
constexpr int RS_NT = 256;
constexpr int RS_RPB = RECD_RS_RPB;  // rows per block (long rows)
// short rows: more rows per block (RECD_RS_SHORT=1), so a block still streams ~16 KB of values
// (a 256-row block of length-8 rows is one 8-value load per thread, all
// latency); the class of a group is chosen from its average row length.  A/B: dedup
// 0.71 ms with the classes vs 0.65 without (the 256-row blocks keep more CTAs
// resident), so it is off.
#ifndef RECD_RS_SHORT
#define RECD_RS_SHORT 0
#endif
constexpr int RS_IT = RECD_RS_IT;    // consecutive values per thread
// uniform chunks stream their values through shared memory with TMA bulk
// copies (3 stages of RT_T values, one thread issues, mbarrier completion):
// every value is read from HBM once, the predecessor row comes from the same
// or the previous stage, and the loads are in flight 2 tiles ahead.  Exact
// (113 dedup/step/fullsize tests green with it on) but slower: row scan 0.465
// vs 0.395 ms, dedup 0.68 vs 0.61 ms (profiles/r2_rowscan_tma_ab.txt); off.
#ifndef RECD_RS_TMA
#define RECD_RS_TMA 0
#endif
// uniform chunks: warp-coalesced 16-byte value pairs (RECD_RS_COAL=1) instead
// of 8 thread-contiguous values per thread
#ifndef RECD_RS_COAL
#define RECD_RS_COAL 1
#endif
constexpr int RT_T = 2048;                                  // values per stage (16 KB)
constexpr int RT_SMEM = RECD_RS_TMA ? 3 * RT_T * 8 : 0;       // dynamic shared memory

#ifndef RECD_RS_SMALLB
#define RECD_RS_SMALLB 1
#endif
#ifndef RECD_RS_MINB
#define RECD_RS_MINB 4
#endif
template <int RS_RPB>
__global__ void __launch_bounds__(RS_NT, RECD_RS_MINB) k_rowscan(const __grid_constant__ DedupParams p) {
  RECD_PDL_PROLOGUE();
  const int g = p.rs_group[blockIdx.y];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * RS_RPB;
  if (r0 >= p.B) return;
  const int64_t r1 = min(p.B, r0 + (int64_t)RS_RPB);
  const int n = (int)(r1 - r0);

  __shared__ int64_t s_start[RS_RPB + 1];
  __shared__ int32_t s_len[RS_RPB];
  __shared__ uint32_t s_mism[RS_RPB];
  __shared__ int s_hashG;  // lanes per head row in the hash pass (32: warp per row)
#if RECD_RS_TMA
  extern __shared__ __align__(128) int64_t s_stage[];  // [3][RT_T]
  __shared__ __align__(8) uint64_t s_bar[3];
  uint32_t tiles_seen = 0;  // staged tiles of earlier features: tile sequence number base
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init1(&s_bar[b]);
    mbar_fence_init();
  }
#endif

  {  // clear this block's slice of the group's hash table
    const int64_t lo = r0 * p.C / p.B, hi = r1 * p.C / p.B;
    unsigned long long* tk = p.tkeys + (int64_t)g * p.C;
    uint32_t* tr = p.treps + (int64_t)g * p.C;
    for (int64_t s = lo + tid; s < hi; s += RS_NT) {
      tk[s] = 0ull;
      tr[s] = 0xffffffffu;
    }
  }
  for (int j = tid; j < n; j += RS_NT) s_mism[j] = (r0 + j == 0) ? 1u : 0u;
  __syncthreads();

  const int fbeg = p.group_first[g], fend = p.group_first[g + 1];
  for (int f = fbeg; f < fend; ++f) {
    const int64_t* off = p.offsets[f];
    const int64_t* val = p.values[f];
    const int64_t nv = nval(p, f);
    for (int j = tid; j <= n; j += RS_NT) {
      const int64_t i = r0 + j;
      s_start[j] = (i < p.B) ? off[i] : nv;
    }
    __syncthreads();
    for (int j = tid; j < n; j += RS_NT) {
      const int64_t i = r0 + j;
      const int64_t len = s_start[j + 1] - s_start[j];
      const int64_t plen = (i > 0) ? (s_start[j] - (j > 0 ? s_start[j - 1] : off[i - 1])) : -1;
      if (plen != len) s_mism[j] = 1u;
      s_len[j] = (int32_t)min(len, (int64_t)INT32_MAX);
    }
    const int64_t vbeg = s_start[0], vend = s_start[n];
    const int64_t tb0 = vbeg & ~(int64_t)(RS_IT - 1);  // 64-byte aligned tiles
    const bool a16 = (reinterpret_cast<uintptr_t>(val) & 15) == 0;
    // uniform-length chunk (every row of a fixed-length history feature): the
    // predecessor of value q is value q - L and its row is (q - vbeg) / L, so
    // no per-value row search; rows whose length differs from the previous
    // row's are already heads, and compares can only set flags, so the chunk's
    // first row needs no special case
    const int64_t L0 = s_start[1] - s_start[0];
    bool uni = L0 > 0 && L0 < (int64_t)(1u << 31) / RS_RPB;  // (q - vbeg) fits 32 bits
    for (int j = tid; j < n; j += RS_NT) uni &= (int64_t)s_len[j] == L0;
    if (tid == 0) s_hashG = 32;
    if (__syncthreads_and(uni)) {
      const uint32_t L = (uint32_t)L0;
      if (tid == 0 && fbeg + 1 == fend && L0 < 32) {
        int G = 1;
        while (G < L0) G <<= 1;
        s_hashG = G;
      }
#if RECD_RS_TMA
      if (a16 && L0 <= RT_T) {
        // tiles [tbeg + t RT_T, +RT_T) of the chunk's values, 16-byte aligned;
        // the copied part of a tile ends at an even value <= vend, a last odd
        // value is read from global memory
        const int64_t tbeg = vbeg & ~(int64_t)1;
        const int ntiles = (int)ceil_div(vend - tbeg, (int64_t)RT_T);
        // tile t is the block's (tiles_seen + t)-th staged tile: stage and
        // barrier (that % 3), barrier phase parity (that / 3) & 1
        auto issue = [&](int t) {
          const int64_t a = tbeg + (int64_t)t * RT_T;
          const int64_t e = min(a + (int64_t)RT_T, vend) & ~(int64_t)1;
          const uint32_t sq = tiles_seen + (uint32_t)t;
          bulk_load(s_stage + (sq % 3) * RT_T, val + a, (uint32_t)(max(e - a, (int64_t)0) * 8),
                    &s_bar[sq % 3]);
        };
        if (tid == 0) {
          issue(0);
          if (ntiles > 1) issue(1);
        }
        const uint32_t dj = RS_NT / L, dr = RS_NT % L;
        for (int t = 0; t < ntiles; ++t) {
          const uint32_t sq = tiles_seen + (uint32_t)t;
          const int b = (int)(sq % 3);
          mbar_wait_parity(&s_bar[b], (sq / 3) & 1u);
          const int64_t a = tbeg + (int64_t)t * RT_T;
          const int64_t ecp = min(a + (int64_t)RT_T, vend) & ~(int64_t)1;  // copied part
          const int64_t* cur = s_stage + b * RT_T;
          const int64_t* prv = s_stage + ((sq + 2) % 3) * RT_T;           // tile t - 1
          // values q = a + k * RS_NT + tid (consecutive threads, consecutive
          // values: conflict-free shared loads); row stepped incrementally
          const int64_t q_first = a + tid;
          uint32_t j = 0, rem = 0;
          if (q_first >= vbeg) {
            const uint32_t rel = (uint32_t)(q_first - vbeg);
            j = rel / L;
            rem = rel - j * L;
          } else {  // only in the first tile, before the chunk's first value
            const uint32_t back = (uint32_t)(vbeg - q_first);  // 1 (tbeg = vbeg - 1)
            rem = L - back;   // the position just before row 0 (skipped below)
            j = 0;
          }
#pragma unroll 4
          for (int k = 0; k < RT_T / RS_NT; ++k) {
            const int64_t q = q_first + (int64_t)k * RS_NT;
            if (q >= vbeg && q < vend) {
              const int64_t v = q < ecp ? cur[q - a] : __ldg(val + q);
              const int64_t pq = q - L0;
              int64_t pv;
              if (pq >= a) pv = cur[pq - a];
              else if (t > 0 && pq >= a - RT_T) pv = prv[pq - (a - RT_T)];
              else pv = __ldg(val + max(pq, (int64_t)0));
              if (pv != v) s_mism[j] = 1u;
            }
            if (q >= vbeg) {
              j += dj;
              rem += dr;
              if (rem >= L) {
                rem -= L;
                ++j;
              }
            } else {   // q = vbeg - 1: the next value of this thread is vbeg - 1 + RS_NT
              const uint32_t rel = (uint32_t)(q + RS_NT - vbeg);
              j = rel / L;
              rem = rel - j * L;
            }
          }
          __syncthreads();  // every thread is done with tile t - 1's stage
          if (tid == 0 && t + 2 < ntiles) issue(t + 2);
        }
        tiles_seen += (uint32_t)ntiles;
        continue;
      }
#endif
#if RECD_RS_COAL
      if (a16) {
        // warp-coalesced: value pair (q, q + 1) of thread tid at q = base + 2 tid
        // + k 512 (consecutive threads, consecutive 16 bytes: 4 L1 lines per
        // warp load instead of 16 for thread-contiguous runs); the predecessor
        // pair at q - L is 16-byte aligned when L is even
        constexpr int PK = RS_IT / 2;                  // pairs per thread per trip
        constexpr int64_t STEP = 2 * RS_NT;            // values per pair slot
        const int64_t tbe = vbeg & ~(int64_t)1;
        const bool Leven = (L & 1u) == 0;
        // rows of a thread's pairs: one division per trip, then stepped by
        // STEP values (dj rows + dr positions) -- ncu: the per-pair division
        // was 12% of the kernel's instructions
        const uint32_t dj = (uint32_t)STEP / L, dr = (uint32_t)STEP % L;
        for (int64_t ob = tbe; ob < vend; ob += STEP * PK) {
          longlong2 cv[PK], pv[PK];
#pragma unroll
          for (int k = 0; k < PK; ++k) {
            const int64_t q = ob + k * STEP + 2 * tid;
            cv[k] = make_longlong2(0, 0);
            if (q + 1 < nv) cv[k] = __ldg(reinterpret_cast<const longlong2*>(val + q));
            else if (q < nv) cv[k].x = __ldg(val + q);
          }
          if (Leven) {  // block-uniform; pq < 0 only in global row 0 (a head anyway)
#pragma unroll
            for (int k = 0; k < PK; ++k) {
              const int64_t pq = ob + k * STEP + 2 * tid - L0;
              pv[k] = __ldg(reinterpret_cast<const longlong2*>(val + (pq < 0 ? 0 : pq)));
            }
          } else {
#pragma unroll
            for (int k = 0; k < PK; ++k) {
              const int64_t pq = ob + k * STEP + 2 * tid - L0;
              pv[k].x = __ldg(val + (pq < 0 ? 0 : pq));
              pv[k].y = __ldg(val + (pq + 1 < 0 ? 0 : pq + 1));
            }
          }
          // q = vbeg - 1 (thread 0's first pair when vbeg is odd): only its
          // second value is in the chunk (row 0); rows from the next pair on
          const int64_t rel0 = ob + 2 * tid - vbeg;
          const bool neg = rel0 < 0;
          uint32_t j, rem;
          {
            const uint32_t r = (uint32_t)(neg ? rel0 + STEP : rel0);
            j = r / L;
            rem = r - j * L;
          }
#pragma unroll
          for (int k = 0; k < PK; ++k) {
            const int64_t q = ob + k * STEP + 2 * tid;
            if (k == 0 && neg) {
              if (cv[k].y != pv[k].y) s_mism[0] = 1u;
              continue;
            }
            if (q < vend) {
              if (cv[k].x != pv[k].x) s_mism[j] = 1u;
              if (q + 1 < vend && cv[k].y != pv[k].y) s_mism[j + (rem + 1 == L ? 1u : 0u)] = 1u;
            }
            j += dj;
            rem += dr;
            if (rem >= L) {
              rem -= L;
              ++j;
            }
          }
        }
        __syncthreads();
        continue;
      }
#endif
      for (int64_t tb = tb0; tb < vend; tb += (int64_t)RS_NT * RS_IT) {
        const int64_t q0 = tb + (int64_t)tid * RS_IT;
        if (q0 >= vend || q0 + RS_IT <= vbeg) continue;
        int64_t v[RS_IT], pv[RS_IT];
        const int64_t pq0 = q0 - L0;
        if (q0 + RS_IT <= nv && a16) {
          const longlong2* src = reinterpret_cast<const longlong2*>(val + q0);
#pragma unroll
          for (int k = 0; k < RS_IT / 2; ++k) {
            const longlong2 t = __ldg(src + k);
            v[2 * k] = t.x;
            v[2 * k + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int k = 0; k < RS_IT; ++k) v[k] = (q0 + k < nv) ? __ldg(val + q0 + k) : 0;
        }
        if (a16 && pq0 >= 0 && (pq0 & 1) == 0) {
          const longlong2* src = reinterpret_cast<const longlong2*>(val + pq0);
#pragma unroll
          for (int k = 0; k < RS_IT / 2; ++k) {
            const longlong2 t = __ldg(src + k);
            pv[2 * k] = t.x;
            pv[2 * k + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int k = 0; k < RS_IT; ++k) pv[k] = __ldg(val + max(pq0 + k, (int64_t)0));
        }
        // row of q0 relative to the chunk (q0 may precede vbeg by < 8)
        const int64_t rel0 = q0 - vbeg;
        uint32_t j = rel0 >= 0 ? (uint32_t)rel0 / L : 0u;
        uint32_t rem = rel0 >= 0 ? (uint32_t)rel0 - j * L : 0u;
#pragma unroll
        for (int k = 0; k < RS_IT; ++k) {
          const int64_t q = q0 + k;
          if (q >= vbeg && q < vend) {
            if (pv[k] != v[k]) s_mism[j] = 1u;
            if (++rem == L) {
              rem = 0;
              ++j;
            }
          }
        }
      }
      __syncthreads();
      continue;
    }
    for (int64_t tb = tb0; tb < vend; tb += (int64_t)RS_NT * RS_IT) {
      const int64_t q0 = tb + (int64_t)tid * RS_IT;
      if (q0 >= vend || q0 + RS_IT <= vbeg) continue;
      int64_t v[RS_IT];
      if (q0 + RS_IT <= nv && a16) {
        const longlong2* src = reinterpret_cast<const longlong2*>(val + q0);
#pragma unroll
        for (int k = 0; k < RS_IT / 2; ++k) {
          const longlong2 t = __ldg(src + k);
          v[2 * k] = t.x;
          v[2 * k + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < RS_IT; ++k) v[k] = (q0 + k < nv) ? __ldg(val + q0 + k) : 0;
      }
      const int64_t qs = max(q0, vbeg);
      int lo = 0, hi = n - 1;  // row containing qs: last j with s_start[j] <= qs
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_start[mid] <= qs) lo = mid; else hi = mid - 1;
      }
      // row of every value, then all predecessor loads, then the compares
      int jk[RS_IT];
      int j = lo;
      int64_t jend = s_start[j + 1];
#pragma unroll
      for (int k = 0; k < RS_IT; ++k) {
        const int64_t q = q0 + k;
        jk[k] = -1;
        if (q >= vbeg && q < vend) {
          while (q >= jend) jend = s_start[++j + 1];
          jk[k] = j;
        }
      }
      int64_t pv[RS_IT];
      const int64_t pq0 = q0 - (int64_t)s_len[max(jk[0], 0)];
      if (a16 && jk[0] >= 0 && jk[0] == jk[RS_IT - 1] && pq0 >= 0 && (pq0 & 1) == 0) {
        // all 8 values in one row of even length: the predecessor's 8 values
        // are contiguous and 16-byte aligned -> 4 vector loads instead of 8
        const longlong2* src = reinterpret_cast<const longlong2*>(val + pq0);
#pragma unroll
        for (int k = 0; k < RS_IT / 2; ++k) {
          const longlong2 t = __ldg(src + k);
          pv[2 * k] = t.x;
          pv[2 * k + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < RS_IT; ++k)
          pv[k] = (jk[k] >= 0) ? __ldg(val + max(q0 + k - (int64_t)s_len[jk[k]], (int64_t)0)) : 0;
      }
#pragma unroll
      for (int k = 0; k < RS_IT; ++k)
        if (jk[k] >= 0 && pv[k] != v[k]) s_mism[jk[k]] = 1u;
    }
    __syncthreads();
  }
  uint8_t* head = p.head + (int64_t)g * p.B;
  for (int j = tid; j < n; j += RS_NT) head[r0 + j] = s_mism[j] ? 1 : 0;
  // content hash of the chunk's heads (their values were just streamed, so
  // the re-read is mostly served by L2).  A single-feature group whose rows
  // share one length L hashes 32 / G rows per warp at once (G = lanes per row,
  // the power of two >= L, <= 32); otherwise a warp per head row, lane-strided.
  const int warp = tid >> 5, lane = tid & 31;
  uint64_t* hash = p.hash + (int64_t)g * p.B;
  const int G = s_hashG;
  if (G < 32) {
    const int gid = lane / G, gl = lane % G, per = 32 / G;
    const int64_t* off = p.offsets[fbeg];
    const int64_t* val0 = p.values[fbeg];
    for (int j0 = warp * per; j0 < n; j0 += (RS_NT / 32) * per) {  // warp-uniform trips
      const int j = j0 + gid;
      const bool mine = j < n && s_mism[j];
      uint64_t h = 0;
      if (mine) {
        const int64_t st = s_start[j];
        const int64_t len = s_start[j + 1] - st;   // == L <= G
        if (gl == 0) h += len_hash(len, 0);
        if (gl < len) h += elem_hash(__ldg(val0 + st + gl), gl, 0);
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1)
        if (d < G) h += __shfl_xor_sync(0xffffffffu, h, d);
      if (mine && gl == 0) hash[r0 + j] = finalize_hash(h, p.hash_mask);
    }
    return;
  }
  for (int j = warp; j < n; j += RS_NT / 32) {
    if (!s_mism[j]) continue;
    const int64_t row = r0 + j;
    uint64_t h = 0;
    for (int f = fbeg; f < fend; ++f) {
      const int fi = f - fbeg;
      const int64_t* off = p.offsets[f];
      const int64_t st = (f == fend - 1) ? s_start[j] : off[row];
      const int64_t len = (f == fend - 1) ? s_start[j + 1] - st : row_end(off, row, p.B, nval(p, f)) - st;
      const int64_t* val = p.values[f] + st;
      if (lane == 0) h += len_hash(len, fi);
      for (int64_t k0 = 0; k0 < len; k0 += 128) {
        int64_t x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t k = k0 + u * 32 + lane;
          x[u] = (k < len) ? __ldg(val + k) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t k = k0 + u * 32 + lane;
          if (k < len) h += elem_hash(x[u], k, fi);
        }
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) h += __shfl_xor_sync(0xffffffffu, h, d);
    if (lane == 0) hash[row] = finalize_hash(h, p.hash_mask);
  }
}

// ----------------------------------------------------------------- insert
// heads only: open-addressing table (64-bit key, L2 resident),
// rep = atomicMin(row) per key -> deterministic min row.
__global__ void __launch_bounds__(256) k_insert(const __grid_constant__ DedupParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.G * p.B) return;
  const int g = (int)(idx / p.B);
  if (!p.head[idx]) return;
  const int64_t i = idx - (int64_t)g * p.B;
  const unsigned long long h = p.hash[idx];
  unsigned long long* tk = p.tkeys + (int64_t)g * p.C;
  uint32_t* tr = p.treps + (int64_t)g * p.C;
  const uint64_t m = (uint64_t)p.C - 1;
  uint64_t s = (h ^ (h >> 29)) & m;
  while (true) {
    const unsigned long long k = atomicCAS(&tk[s], 0ull, h);
    if (k == 0ull || k == h) {
      atomicMin(&tr[s], (uint32_t)i);
      p.slot_of[idx] = (uint32_t)s;
      return;
    }
    s = (s + 1) & m;
  }
}

// ---------------------------------------------------------------- resolve
__global__ void __launch_bounds__(256) k_resolve(const __grid_constant__ DedupParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.G * p.B) return;
  if (!p.head[idx]) return;
  const int g = (int)(idx / p.B);
  const int64_t i = idx - (int64_t)g * p.B;
  const int64_t r = p.treps[(int64_t)g * p.C + p.slot_of[idx]];
  if (r == i) {
    p.cls[idx] = (int32_t)i;
  } else if (rows_equal(p, g, i, r)) {
    p.cls[idx] = (int32_t)r;
  } else {
    p.cls[idx] = -1;  // hash collision with a different row: exact fallback
    p.collide[g] = 1;
  }
}

// --------------------------------------------------------------- fallback
// Pending heads (content differs from their slot's min row) are resolved in
// ascending row order against the secondary representatives created so far;
// the first row of each content class becomes its representative, as the
// reference's bucket scan does (tensors.py:288-297).
constexpr int FB_NT = 256;
__global__ void __launch_bounds__(FB_NT) k_fallback(const __grid_constant__ DedupParams p) {
  RECD_PDL_PROLOGUE();
  const int g = blockIdx.x;
  if (!p.collide[g]) return;
  const int tid = threadIdx.x;
  const uint8_t* head = p.head + (int64_t)g * p.B;
  const uint64_t* hash = p.hash + (int64_t)g * p.B;
  int32_t* cls = p.cls + (int64_t)g * p.B;
  int32_t* list = p.fb_list + (int64_t)g * p.B;
  __shared__ int64_t s_scan[32];
  __shared__ int32_t s_pend[FB_NT];
  __shared__ int s_np;
  __shared__ int s_found;
  int nl = 0;  // uniform across the block
  for (int64_t base = 0; base < p.B; base += FB_NT) {
    const int64_t i = base + tid;
    const bool pend = i < p.B && head[i] && cls[i] == -1;
    int64_t tot;
    const int64_t pos = block_exclusive_scan<FB_NT>(pend ? 1 : 0, s_scan, &tot);
    if (pend) s_pend[pos] = (int32_t)i;
    if (tid == 0) s_np = (int)tot;
    __syncthreads();
    const int np = s_np;
    for (int k = 0; k < np; ++k) {
      const int64_t row = s_pend[k];
      const uint64_t h = hash[row];
      if (tid == 0) s_found = 0x7fffffff;
      __syncthreads();
      for (int e = tid; e < nl; e += FB_NT) {
        const int32_t q = list[e];
        if (hash[q] == h && rows_equal(p, g, row, q)) atomicMin(&s_found, q);
      }
      __syncthreads();
      const int found = s_found;
      if (tid == 0) {
        if (found != 0x7fffffff) {
          cls[row] = found;
        } else {
          cls[row] = (int32_t)row;
          list[nl] = (int32_t)row;
        }
      }
      if (found == 0x7fffffff) ++nl;
      __syncthreads();
    }
  }
}

// ----------------------------------------------------------------- number
// Chunk-parallel numbering (2048-row chunks): a row is a first occurrence iff
// it is a head that represents its class (cls[i] == i), which is known
// locally, so numbering is reduce -> scan -> downsweep:
//   k_num_reduce  per chunk: last head, #first rows, their value counts per feature
//   k_num_scan    per group: exclusive chunk prefixes (+ incoming run head), totals
//   k_num_down    per chunk: run-head propagation (cls of every row), uid of
//                 first rows, first_rows[uid], unique offsets per feature
//   k_num_inv     inverse[i] = uidmap[cls[i]] (needs every chunk's uidmap)
constexpr int NB_NT = 256;
constexpr int NB_ITEMS = 8;              // rows per thread (big batches: 2048-row chunks)
#ifndef RECD_NB_SMALL
#define RECD_NB_SMALL 1
#endif
constexpr int NB_ITEMS_SMALL = 1;        // small batches (< 32,768 rows): 256-row chunks,
                                         // 8x the blocks of a latency-bound numbering

template <int NB_ITEMS>
__global__ void __launch_bounds__(NB_NT) k_num_reduce(const __grid_constant__ DedupParams p) {
  constexpr int NB_CH = NB_NT * NB_ITEMS;
  RECD_PDL_PROLOGUE();
  const int g = blockIdx.y;
  const int64_t c = blockIdx.x;
  const int64_t B = p.B;
  const int tid = threadIdx.x;
  const uint8_t* head = p.head + (int64_t)g * B;
  const int32_t* cls = p.cls + (int64_t)g * B;
  const int64_t i0 = c * NB_CH + (int64_t)tid * NB_ITEMS;
  __shared__ int64_t s_scan[32];
  int64_t lrh = -1, nf = 0;
  bool first[NB_ITEMS];
#pragma unroll
  for (int k = 0; k < NB_ITEMS; ++k) {
    const int64_t i = i0 + k;
    first[k] = false;
    if (i < B && head[i]) {
      lrh = i;
      first[k] = cls[i] == (int32_t)i;
      nf += first[k];
    }
  }
  const int64_t nch = ceil_div(B, NB_CH);
  int64_t tot;
  block_inclusive_max<NB_NT>(lrh, s_scan, &tot);
  if (tid == 0) p.nb_rh[(int64_t)g * nch + c] = tot;
  block_exclusive_scan<NB_NT>(nf, s_scan, &tot);
  if (tid == 0) p.nb_nf[(int64_t)g * nch + c] = tot;
  for (int f = p.group_first[g]; f < p.group_first[g + 1]; ++f) {
    const int64_t* off = p.offsets[f];
    int64_t ls = 0;
#pragma unroll
    for (int k = 0; k < NB_ITEMS; ++k)
      if (first[k]) ls += row_end(off, i0 + k, B, nval(p, f)) - off[i0 + k];
    block_exclusive_scan<NB_NT>(ls, s_scan, &tot);
    if (tid == 0) p.nb_len[(int64_t)f * nch + c] = tot;
  }
}

// block per group: chunk prefixes in place (rh -> incoming run head, an
// exclusive max; nf / len -> exclusive sums) and the group's totals
__global__ void __launch_bounds__(NB_NT) k_num_scan(const __grid_constant__ DedupParams p) {
  RECD_PDL_PROLOGUE();
  const int g = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t nch = ceil_div(p.B, (int64_t)p.nb_ch);
  __shared__ int64_t s_scan[32];
  __shared__ int64_t s_last[NB_NT];
  int64_t crh = -1, cnf = 0;
  for (int64_t c0 = 0; c0 < nch; c0 += NB_NT) {
    const int64_t c = c0 + tid;
    int64_t* rh = p.nb_rh + (int64_t)g * nch;
    int64_t* nf = p.nb_nf + (int64_t)g * nch;
    const int64_t vrh = c < nch ? rh[c] : -1;
    const int64_t vnf = c < nch ? nf[c] : 0;
    int64_t tot;
    const int64_t incl = block_inclusive_max<NB_NT>(vrh, s_scan, &tot);
    s_last[tid] = incl;
    __syncthreads();
    const int64_t excl = max(crh, tid ? s_last[tid - 1] : (int64_t)-1);
    __syncthreads();
    crh = max(crh, tot);
    const int64_t x = block_exclusive_scan<NB_NT>(vnf, s_scan, &tot);
    if (c < nch) {
      rh[c] = excl;
      nf[c] = cnf + x;
    }
    cnf += tot;
  }
  for (int f = p.group_first[g]; f < p.group_first[g + 1]; ++f) {
    int64_t* ln = p.nb_len + (int64_t)f * nch;
    int64_t carry = 0;
    for (int64_t c0 = 0; c0 < nch; c0 += NB_NT) {
      const int64_t c = c0 + tid;
      int64_t tot;
      const int64_t x = block_exclusive_scan<NB_NT>(c < nch ? ln[c] : 0, s_scan, &tot);
      if (c < nch) ln[c] = carry + x;
      carry += tot;
    }
    if (tid == 0) {
      p.count_rows[f] = cnf;
      p.count_vals[f] = carry;
    }
  }
}

template <int NB_ITEMS>
__global__ void __launch_bounds__(NB_NT) k_num_down(const __grid_constant__ DedupParams p) {
  constexpr int NB_CH = NB_NT * NB_ITEMS;
  RECD_PDL_PROLOGUE();
  const int g = blockIdx.y;
  const int64_t c = blockIdx.x;
  const int64_t B = p.B;
  const int tid = threadIdx.x;
  const int64_t nch = ceil_div(B, NB_CH);
  const uint8_t* head = p.head + (int64_t)g * B;
  int32_t* cls = p.cls + (int64_t)g * B;
  int32_t* uidmap = p.uidmap + (int64_t)g * B;
  int32_t* first_rows = p.first_rows + (int64_t)g * B;
  const int64_t i0 = c * NB_CH + (int64_t)tid * NB_ITEMS;
  __shared__ int64_t s_scan[32];
  __shared__ int64_t s_last[NB_NT];
  // run heads: exclusive max over the chunk's threads, seeded with the incoming head
  int64_t lrh = -1;
  bool hd[NB_ITEMS];
#pragma unroll
  for (int k = 0; k < NB_ITEMS; ++k) {
    const int64_t i = i0 + k;
    hd[k] = i < B && head[i];
    if (hd[k]) lrh = i;
  }
  int64_t tot;
  const int64_t incl = block_inclusive_max<NB_NT>(lrh, s_scan, &tot);
  s_last[tid] = incl;
  __syncthreads();
  int64_t rh = max(p.nb_rh[(int64_t)g * nch + c], tid ? s_last[tid - 1] : (int64_t)-1);
  bool first[NB_ITEMS];
  int64_t nf = 0;
#pragma unroll
  for (int k = 0; k < NB_ITEMS; ++k) {
    const int64_t i = i0 + k;
    first[k] = false;
    if (i < B) {
      if (hd[k]) {
        rh = i;
        first[k] = cls[i] == (int32_t)i;
        nf += first[k];
      } else {
        cls[i] = cls[rh];  // rh is a head: its cls is final and never rewritten
      }
    }
  }
  int64_t uid = p.nb_nf[(int64_t)g * nch + c] + block_exclusive_scan<NB_NT>(nf, s_scan, &tot);
  int64_t uids[NB_ITEMS];
#pragma unroll
  for (int k = 0; k < NB_ITEMS; ++k) {
    uids[k] = uid;
    if (first[k]) {
      uidmap[i0 + k] = (int32_t)uid;
      first_rows[uid] = (int32_t)(i0 + k);
      ++uid;
    }
  }
  for (int f = p.group_first[g]; f < p.group_first[g + 1]; ++f) {
    const int64_t* off = p.offsets[f];
    int64_t len[NB_ITEMS];
    int64_t ls = 0;
#pragma unroll
    for (int k = 0; k < NB_ITEMS; ++k) {
      len[k] = first[k] ? row_end(off, i0 + k, B, nval(p, f)) - off[i0 + k] : 0;
      ls += len[k];
    }
    int64_t o = p.nb_len[(int64_t)f * nch + c] + block_exclusive_scan<NB_NT>(ls, s_scan, &tot);
    int64_t* uoff = p.uoffsets[f];
#pragma unroll
    for (int k = 0; k < NB_ITEMS; ++k)
      if (first[k]) {
        uoff[uids[k]] = o;
        o += len[k];
      }
  }
}

__global__ void __launch_bounds__(256) k_num_inv(const __grid_constant__ DedupParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.G * p.B) return;
  const int g = (int)(idx / p.B);
  p.inverse[g][idx - (int64_t)g * p.B] = p.uidmap[(int64_t)g * p.B + p.cls[idx]];
}

// ------------------------------------------------------------------- copy
// Value-parallel gather of the unique lists: block per 4096 unique values of
// a feature.  The block locates its first unique row (32-ary warp search over
// the unique offsets), stages (unique offset, source offset) of the rows it
// spans in shared memory with one independent load chain per row, then the
// block copies the values with consecutive threads on consecutive values.
constexpr int CP_NT = 256;
#ifndef RECD_CP_IT
#define RECD_CP_IT 64
#endif
#ifndef RECD_TINY_CH  // 1K unique values per k_copy block on tiny batches
#define RECD_TINY_CH 1
#endif
constexpr int CP_IT = RECD_CP_IT;
#ifndef RECD_CP_ILP  // gathers in flight per thread in the uniform-row copy
#define RECD_CP_ILP 4
#endif
constexpr int CP_ILP = RECD_CP_ILP;
constexpr int CP_CH = CP_NT * CP_IT;  // unique values per block
constexpr int CP_MAXR = 512;          // rows staged per pass


__global__ void __launch_bounds__(CP_NT) k_copy(const __grid_constant__ DedupParams p) {
  RECD_PDL_PROLOGUE();
  const int f = block_feature(p.cp_blk0, p.F, (int64_t)blockIdx.x);
  const int64_t j0 = ((int64_t)blockIdx.x - p.cp_blk0[f]) * p.cp_ch;
  const int64_t U = p.count_rows[f], NV = p.count_vals[f];
  if (j0 >= NV) return;
  const int64_t j1 = min(NV, j0 + p.cp_ch);
  const int tid = threadIdx.x;
  const int64_t* uoff = p.uoffsets[f];
  const int64_t* off = p.offsets[f];
  const int64_t* src = p.values[f];
  int64_t* dst = p.uvalues[f];
  int64_t* rdst = p.rdst[f] ? p.rdst[f] + *p.rbase[f] : nullptr;
  const int32_t* frows = p.first_rows + (int64_t)p.feat_group[f] * p.B;
  __shared__ int64_t s_u0;
  __shared__ int64_t s_uo[CP_MAXR + 1];
  __shared__ int64_t s_so[CP_MAXR];
  if (tid < 32) {
    const int64_t u = warp_last_le(uoff, U, j0, tid);
    if (tid == 0) s_u0 = u;
  }
  __syncthreads();
  int64_t u0 = s_u0;
  while (true) {
    const int nr = (int)min((int64_t)CP_MAXR, U - u0);
    for (int t = tid; t <= nr; t += CP_NT) {
      const int64_t u = u0 + t;
      s_uo[t] = (t < nr) ? uoff[u] : ((u < U) ? uoff[u] : NV);
      if (t < nr) s_so[t] = off[frows[u]];
    }
    __syncthreads();
    const int64_t covered = s_uo[nr];  // values before row u0 + nr
    const int64_t qa = max(j0, s_uo[0]), qb = min(j1, covered);
    // staged rows all of one length L (fixed-length history features): the row
    // of value q is (q - s_uo[0]) / L, stepped incrementally; loads batched 4
    // deep so every thread keeps 4 independent gathers in flight
    const int64_t L0 = nr > 0 ? s_uo[1] - s_uo[0] : 0;
    bool uni = L0 > 0 && L0 < (1 << 23);
    for (int t = tid; t < nr; t += CP_NT) uni &= (s_uo[t + 1] - s_uo[t]) == L0;
    if (__syncthreads_and(uni)) {
      const uint32_t L = (uint32_t)L0, dj = CP_NT / L, dr = CP_NT % L;
      const int64_t q_first = qa + tid;
      uint32_t r = 0, rem = 0;
      if (q_first < qb) {
        const uint32_t rel = (uint32_t)(q_first - s_uo[0]);
        r = rel / L;
        rem = rel - r * L;
      }
      for (int64_t qq = q_first; qq < qb; qq += CP_ILP * CP_NT) {
        int64_t a[CP_ILP], v[CP_ILP];
#pragma unroll
        for (int k = 0; k < CP_ILP; ++k) {
          a[k] = s_so[min(r, (uint32_t)(nr - 1))] + rem;
          r += dj;
          rem += dr;
          if (rem >= L) {
            rem -= L;
            ++r;
          }
        }
#pragma unroll
        for (int k = 0; k < CP_ILP; ++k)
          if (qq + k * CP_NT < qb) v[k] = __ldg(src + a[k]);
#pragma unroll
        for (int k = 0; k < CP_ILP; ++k) {
          const int64_t q = qq + k * CP_NT;
          if (q < qb) {
            dst[q] = v[k];
            if (rdst) rdst[q] = v[k];
          }
        }
      }
      if (covered >= j1) break;
      __syncthreads();
      u0 += nr;
      continue;
    }
    // values qa + k * CP_NT + tid: coalesced loads and stores; the row of each
    // value by a search over the staged rows, starting from the previous one
    int r = 0;
    for (int64_t q = qa + tid; q < qb; q += CP_NT) {
      // row of q: short forward walk from the previous value's row (q moved
      // by one block stride), binary search only past 8 rows
      if (s_uo[min(r + 8, nr)] <= q) {
        int lo = r + 8, hi = nr - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_uo[mid] <= q) lo = mid; else hi = mid - 1;
        }
        r = lo;
      } else {
        while (s_uo[r + 1] <= q) ++r;
      }
      const int64_t v = __ldg(src + s_so[r] + (q - s_uo[r]));
      dst[q] = v;
      if (rdst) rdst[q] = v;
    }
    if (covered >= j1) break;
    __syncthreads();
    u0 += nr;
  }
}

struct DedupScratch {
  uint8_t* head;
  uint64_t* hash;
  uint32_t* slot_of;
  int32_t *cls, *uidmap, *first_rows, *fb_list, *collide;
  int64_t *nb_rh, *nb_nf, *nb_len;
  unsigned long long* tkeys;
  uint32_t* treps;
};

static size_t carve_dedup(void* base, size_t cap, int G, int F, int64_t B, int64_t C,
                          DedupScratch* s) {
  Arena a(base, cap);
  const int64_t nch = ceil_div(B, NB_NT * NB_ITEMS_SMALL);  // the most chunks either layout has
  s->nb_rh = a.take<int64_t>((size_t)G * nch);
  s->nb_nf = a.take<int64_t>((size_t)G * nch);
  s->nb_len = a.take<int64_t>((size_t)F * nch);
  s->head = a.take<uint8_t>((size_t)G * B);
  s->hash = a.take<uint64_t>((size_t)G * B);
  s->slot_of = a.take<uint32_t>((size_t)G * B);
  s->cls = a.take<int32_t>((size_t)G * B);
  s->uidmap = a.take<int32_t>((size_t)G * B);
  s->first_rows = a.take<int32_t>((size_t)G * B);
  s->fb_list = a.take<int32_t>((size_t)G * B);
  s->collide = a.take<int32_t>((size_t)G);
  s->tkeys = a.take<unsigned long long>((size_t)G * C);
  s->treps = a.take<uint32_t>((size_t)G * C);
  return a.used;
}

static int64_t table_slots(int64_t B) { return (int64_t)next_pow2((uint64_t)std::max<int64_t>(2 * B, 64)); }

}  // namespace recd

using namespace recd;

extern "C" void recd_debug_set_hash_mask(uint64_t mask) { g_hash_mask = mask ? mask : ~0ull; }

extern "C" size_t recd_dedup_scratch_bytes(int32_t num_groups, int32_t num_features,
                                           int64_t batch_size) {
  DedupScratch s;
  // groups are processed in chunks of <= RECD_MAX_FEAT features; size for all
  return carve_dedup(nullptr, 0, std::max(num_groups, 1), std::max(num_features, 1), batch_size,
                     table_slots(batch_size), &s);
}

enum { DD_NUMBER = 1, DD_COPY = 2, DD_ALL = 3 };

static int run_dedup(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                     const int64_t* const* values, const int64_t* const* offsets,
                     const int64_t* num_values, int64_t* const* inverse_out,
                     int64_t* const* uoffsets_out, int64_t* const* uvalues_out, int64_t* counts_out,
                     void* scratch, size_t scratch_bytes, cudaStream_t stream, int phase,
                     int64_t* const* remote_values, const int64_t* const* remote_base,
                     const int64_t* num_values_dev = nullptr) {
  if (num_groups <= 0 || batch_size <= 0 || batch_size >= (1ll << 31) || !group_sizes)
    return RECD_ERR_ARG;
  int F = 0;
  for (int g = 0; g < num_groups; ++g) {
    if (group_sizes[g] <= 0 || group_sizes[g] > RECD_MAX_FEAT) return RECD_ERR_ARG;
    F += group_sizes[g];
  }
  const int64_t B = batch_size, C = table_slots(B);
  DedupScratch s;
  if (carve_dedup(scratch, scratch_bytes, num_groups, F, B, C, &s) > scratch_bytes) return RECD_ERR_SCRATCH;
  if (phase & DD_NUMBER)
    RECD_CUDA_CHECK(cudaMemsetAsync(s.collide, 0, sizeof(int32_t) * num_groups, stream));

  int g0 = 0, f0 = 0;
  while (g0 < num_groups) {
    // chunk of consecutive groups with <= RECD_MAX_FEAT features
    int g1 = g0, nf = 0;
    while (g1 < num_groups && nf + group_sizes[g1] <= RECD_MAX_FEAT) nf += group_sizes[g1++];
    DedupParams p;
    memset(&p, 0, sizeof(p));
    p.G = g1 - g0;
    p.F = nf;
    p.B = B;
    p.C = C;
    p.hash_mask = g_hash_mask;
    p.nv_dev = num_values_dev ? num_values_dev + f0 : nullptr;
    int f = 0;
    for (int g = 0; g < p.G; ++g) {
      p.group_first[g] = f;
      p.inverse[g] = inverse_out[g0 + g];
      for (int k = 0; k < group_sizes[g0 + g]; ++k, ++f) {
        p.feat_group[f] = g;
        p.values[f] = values[f0 + f];
        p.offsets[f] = offsets[f0 + f];
        p.nvalues[f] = num_values[f0 + f];
        p.uoffsets[f] = uoffsets_out[f0 + f];
        p.uvalues[f] = uvalues_out[f0 + f];
        p.rdst[f] = remote_values ? remote_values[f0 + f] : nullptr;
        p.rbase[f] = remote_base ? remote_base[f0 + f] : nullptr;
        if (p.rdst[f] && !p.rbase[f]) return RECD_ERR_ARG;
        if (!p.offsets[f] || !p.inverse[g] || !p.uoffsets[f] || (!p.values[f] && p.nvalues[f] > 0))
          return RECD_ERR_ARG;
      }
    }
    p.group_first[p.G] = f;
    p.count_rows = counts_out + f0;
    p.count_vals = counts_out + F + f0;
    p.head = s.head + (int64_t)g0 * B;
    p.hash = s.hash + (int64_t)g0 * B;
    p.slot_of = s.slot_of + (int64_t)g0 * B;
    p.cls = s.cls + (int64_t)g0 * B;
    p.uidmap = s.uidmap + (int64_t)g0 * B;
    p.first_rows = s.first_rows + (int64_t)g0 * B;
    p.fb_list = s.fb_list + (int64_t)g0 * B;
    p.collide = s.collide + g0;
    {
      p.nb_ch = NB_NT * (RECD_NB_SMALL && B < 32768 ? NB_ITEMS_SMALL : NB_ITEMS);
      const int64_t nch = ceil_div(B, (int64_t)p.nb_ch);
      p.nb_rh = s.nb_rh + (int64_t)g0 * nch;
      p.nb_nf = s.nb_nf + (int64_t)g0 * nch;
      p.nb_len = s.nb_len + (int64_t)f0 * nch;
    }
    p.tkeys = s.tkeys + (int64_t)g0 * C;
    p.treps = s.treps + (int64_t)g0 * C;

    const int64_t rows = (int64_t)p.G * B;
    double rs_avg[RECD_MAX_FEAT];
    {  // groups with the most values first (their blocks are the longest)
      std::vector<std::pair<int64_t, int>> order;
      for (int g = 0; g < p.G; ++g) {
        int64_t nvg = 0;
        for (int ff = p.group_first[g]; ff < p.group_first[g + 1]; ++ff) nvg += p.nvalues[ff];
        order.push_back({-nvg, g});
      }
      std::stable_sort(order.begin(), order.end());
      for (int k = 0; k < p.G; ++k) p.rs_group[k] = order[k].second;
      // row-scan class per group by its average row length (values per row)
      for (int k = 0; k < p.G; ++k) rs_avg[k] = (double)(-order[k].first) / (double)B;
    }
    if (phase & DD_NUMBER) {
      {
        // groups are ordered by value count (most first): long-row groups take
        // 256-row blocks, rows of <= 12 values 2048-row blocks, <= 48 1024
        int k0 = 0;
        if (RT_SMEM > 0) {  // opt in to the staged row scan's dynamic shared memory
          static bool attr[64] = {};
          int dev = 0;
          RECD_CUDA_CHECK(cudaGetDevice(&dev));
          if (dev < 0 || dev >= 64 || !attr[dev]) {
            RECD_CUDA_CHECK(cudaFuncSetAttribute(k_rowscan<RS_RPB>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, RT_SMEM));
            RECD_CUDA_CHECK(cudaFuncSetAttribute(k_rowscan<1024>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, RT_SMEM));
            RECD_CUDA_CHECK(cudaFuncSetAttribute(k_rowscan<2048>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, RT_SMEM));
            if (dev >= 0 && dev < 64) attr[dev] = true;
          }
        }
        auto launch_class = [&](int k1, int rpb) {
          if (k1 <= k0) return;
          DedupParams q = p;
          for (int k = k0; k < k1; ++k) q.rs_group[k - k0] = p.rs_group[k];
          const dim3 grid((unsigned)ceil_div(B, rpb), (unsigned)(k1 - k0));
          if (rpb == 64) pdl(k_rowscan<64>, grid, RS_NT, RT_SMEM, stream)(q);
          else if (rpb == 2048) pdl(k_rowscan<2048>, grid, RS_NT, RT_SMEM, stream)(q);
          else if (rpb == 1024) pdl(k_rowscan<1024>, grid, RS_NT, RT_SMEM, stream)(q);
          else pdl(k_rowscan<RS_RPB>, grid, RS_NT, RT_SMEM, stream)(q);
          note_launch();
          k0 = k1;
        };
        int k1 = 0;
        while (k1 < p.G && (!RECD_RS_SHORT || rs_avg[k1] > 48.0)) ++k1;
        // small batches (latency-bound): 64-row blocks, 4x the blocks in flight
        launch_class(k1, (RECD_RS_SMALLB && B < 32768) ? 64 : RS_RPB);
        while (k1 < p.G && rs_avg[k1] > 12.0) ++k1;
        launch_class(k1, 1024);
        launch_class(p.G, 2048);
      }
      pdl(k_insert, (unsigned)ceil_div(rows, 256), 256, 0, stream)(p);
      pdl(k_resolve, (unsigned)ceil_div(rows, 256), 256, 0, stream)(p);
      pdl(k_fallback, p.G, FB_NT, 0, stream)(p);
      const dim3 ng((unsigned)ceil_div(B, (int64_t)p.nb_ch), p.G);
      if (p.nb_ch == NB_NT * NB_ITEMS) {
        pdl(k_num_reduce<NB_ITEMS>, ng, NB_NT, 0, stream)(p);
        pdl(k_num_scan, p.G, NB_NT, 0, stream)(p);
        pdl(k_num_down<NB_ITEMS>, ng, NB_NT, 0, stream)(p);
      } else {
        pdl(k_num_reduce<NB_ITEMS_SMALL>, ng, NB_NT, 0, stream)(p);
        pdl(k_num_scan, p.G, NB_NT, 0, stream)(p);
        pdl(k_num_down<NB_ITEMS_SMALL>, ng, NB_NT, 0, stream)(p);
      }
      pdl(k_num_inv, (unsigned)ceil_div(rows, 256), 256, 0, stream)(p);
      note_launch(7);
    }
    if (phase & DD_COPY) {
      // 16K values per block on big batches (setup amortised), 4K on small
      // ones (more blocks in flight); A/B: dedup 0.67 -> 0.61 ms at cfg2
      int64_t tot = 0;
      for (int ff = 0; ff < p.F; ++ff) tot += p.nvalues[ff];
      p.cp_ch = (int64_t)CP_NT * (tot >= (8ll << 20) ? CP_IT : (tot >= (1ll << 20) || !RECD_TINY_CH) ? 16 : 4);
      int64_t cblk = 0;
      for (int ff = 0; ff < p.F; ++ff) {
        p.cp_blk0[ff] = cblk;
        cblk += std::max<int64_t>(1, ceil_div(p.nvalues[ff], p.cp_ch));
      }
      p.cp_blk0[p.F] = cblk;
      pdl(k_copy, (unsigned)cblk, CP_NT, 0, stream)(p);
      note_launch(1);
    }
    RECD_LAUNCH_CHECK();
    g0 = g1;
    f0 += nf;
  }
  return RECD_OK;
}

extern "C" int recd_dedup(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                          const int64_t* const* values, const int64_t* const* offsets,
                          const int64_t* num_values, int64_t* const* inverse_out,
                          int64_t* const* uoffsets_out, int64_t* const* uvalues_out,
                          int64_t* counts_out, void* scratch, size_t scratch_bytes,
                          recd_stream_t stream) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_groups);
  return run_dedup(num_groups, group_sizes, batch_size, values, offsets, num_values, inverse_out,
                   uoffsets_out, uvalues_out, counts_out, scratch, scratch_bytes,
                   (cudaStream_t)stream, DD_ALL, nullptr, nullptr);
}

// recd_dedup in two halves (same arguments, same scratch): _number computes the
// inverse, unique offsets and counts; _copy gathers the unique values and can
// also store them into a second (peer) buffer at a device-side base -- the
// row-sharded step's ID dispatch fused into the gather.
extern "C" int recd_dedup_number(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                                 const int64_t* const* values, const int64_t* const* offsets,
                                 const int64_t* num_values, int64_t* const* inverse_out,
                                 int64_t* const* uoffsets_out, int64_t* const* uvalues_out,
                                 int64_t* counts_out, void* scratch, size_t scratch_bytes,
                                 recd_stream_t stream) {
  return run_dedup(num_groups, group_sizes, batch_size, values, offsets, num_values, inverse_out,
                   uoffsets_out, uvalues_out, counts_out, scratch, scratch_bytes,
                   (cudaStream_t)stream, DD_NUMBER, nullptr, nullptr);
}

extern "C" int recd_dedup_copy(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                               const int64_t* const* values, const int64_t* const* offsets,
                               const int64_t* num_values, int64_t* const* inverse_out,
                               int64_t* const* uoffsets_out, int64_t* const* uvalues_out,
                               int64_t* counts_out, int64_t* const* remote_values,
                               const int64_t* const* remote_base, void* scratch,
                               size_t scratch_bytes, recd_stream_t stream) {
  return run_dedup(num_groups, group_sizes, batch_size, values, offsets, num_values, inverse_out,
                   uoffsets_out, uvalues_out, counts_out, scratch, scratch_bytes,
                   (cudaStream_t)stream, DD_COPY, remote_values, remote_base);
}

// recd_dedup with the per-feature value counts on the device (num_values_dev,
// int64[F]) and host capacities (value_caps) for the launch geometry: the
// counts of a new batch are written to device memory together with its
// values, so one captured graph serves every batch up to the capacities.
// phase: 1 = number (inverse, unique offsets, counts), 2 = copy (unique values,
// optionally also into remote_values at *remote_base), 3 = both.
extern "C" int recd_dedup_ex(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                             const int64_t* const* values, const int64_t* const* offsets,
                             const int64_t* value_caps, const int64_t* num_values_dev,
                             int32_t phase, int64_t* const* inverse_out,
                             int64_t* const* uoffsets_out, int64_t* const* uvalues_out,
                             int64_t* counts_out, int64_t* const* remote_values,
                             const int64_t* const* remote_base, void* scratch,
                             size_t scratch_bytes, recd_stream_t stream) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_groups);
  if (!num_values_dev || !value_caps || phase < 1 || phase > 3) return RECD_ERR_ARG;
  return run_dedup(num_groups, group_sizes, batch_size, values, offsets, value_caps, inverse_out,
                   uoffsets_out, uvalues_out, counts_out, scratch, scratch_bytes,
                   (cudaStream_t)stream, phase, remote_values, remote_base, num_values_dev);
}
