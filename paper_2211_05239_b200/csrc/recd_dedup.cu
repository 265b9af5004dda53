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
//   k_insert   heads only: warp-cooperative 64-bit row hash, open-addressing
//              table (64-bit key, L2 resident), rep = atomicMin(row) per key.
//   k_resolve  heads whose rep != self are fully compared with the rep; a
//              mismatch (a true 64-bit collision) is marked pending.
//   k_fallback (cold) exact sequential resolution of pending heads.
//   k_number   one CTA per group: run-head propagation, first-occurrence
//              flags, uid scan, inverse, unique offsets (one scan per feature).
//   k_copy     warp per unique row copies its lists into the unique values.
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
  int64_t nvalues[RECD_MAX_FEAT];
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
  int32_t* fb_list;     // [G][B]
  unsigned long long* tkeys;  // [G][C]
  uint32_t* treps;            // [G][C]
  int32_t* collide;           // [G]
  int rs_group[RECD_MAX_FEAT];  // k_rowscan: groups in launch order (most values first)
};

__device__ __forceinline__ int64_t row_begin(const int64_t* off, int64_t i) { return off[i]; }
__device__ __forceinline__ int64_t row_end(const int64_t* off, int64_t i, int64_t B, int64_t nv) {
  return (i + 1 < B) ? off[i + 1] : nv;
}

__device__ bool rows_equal(const DedupParams& p, int g, int64_t a, int64_t b) {
  for (int f = p.group_first[g]; f < p.group_first[g + 1]; ++f) {
    const int64_t* off = p.offsets[f];
    const int64_t* val = p.values[f];
    int64_t sa = off[a], ea = row_end(off, a, p.B, p.nvalues[f]);
    int64_t sb = off[b], eb = row_end(off, b, p.B, p.nvalues[f]);
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
constexpr int RS_NT = 256;
constexpr int RS_RPB = 256;
constexpr int RS_IT = 8;  // consecutive values per thread

__global__ void __launch_bounds__(RS_NT) k_rowscan(const __grid_constant__ DedupParams p) {
  const int g = p.rs_group[blockIdx.y];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * RS_RPB;
  if (r0 >= p.B) return;
  const int64_t r1 = min(p.B, r0 + (int64_t)RS_RPB);
  const int n = (int)(r1 - r0);

  __shared__ int64_t s_start[RS_RPB + 1];
  __shared__ int32_t s_len[RS_RPB];
  __shared__ uint32_t s_mism[RS_RPB];

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
    const int64_t nv = p.nvalues[f];
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
    __syncthreads();
    const int64_t vbeg = s_start[0], vend = s_start[n];
    const int64_t tb0 = vbeg & ~(int64_t)(RS_IT - 1);  // 64-byte aligned tiles
    const bool a16 = (reinterpret_cast<uintptr_t>(val) & 15) == 0;
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
#pragma unroll
      for (int k = 0; k < RS_IT; ++k)
        pv[k] = (jk[k] >= 0) ? __ldg(val + max(q0 + k - (int64_t)s_len[jk[k]], (int64_t)0)) : 0;
#pragma unroll
      for (int k = 0; k < RS_IT; ++k)
        if (jk[k] >= 0 && pv[k] != v[k]) s_mism[jk[k]] = 1u;
    }
    __syncthreads();
  }
  uint8_t* head = p.head + (int64_t)g * p.B;
  for (int j = tid; j < n; j += RS_NT) head[r0 + j] = s_mism[j] ? 1 : 0;
}

// ----------------------------------------------------------------- insert
// Warp per 32 rows of a group: the run heads among them are hashed one at a
// time by the whole warp (lane-strided, coalesced), then every head lane
// inserts its hash: open addressing, rep = atomicMin(row) per key.
__global__ void __launch_bounds__(256) k_insert(const __grid_constant__ DedupParams p) {
  const int64_t wpg = ceil_div(p.B, 32);
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= (int64_t)p.G * wpg) return;
  const int lane = threadIdx.x & 31;
  const int g = (int)(w / wpg);
  const int64_t i = (w - (int64_t)g * wpg) * 32 + lane;
  const int64_t idx = (int64_t)g * p.B + i;
  const bool is_head = i < p.B && p.head[idx];
  unsigned m = __ballot_sync(0xffffffffu, is_head);
  if (!m) return;
  const int fbeg = p.group_first[g], fend = p.group_first[g + 1];
  uint64_t mine = 0;
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int64_t row = i - lane + src;
    uint64_t h = 0;
    for (int f = fbeg; f < fend; ++f) {
      const int fi = f - fbeg;
      const int64_t* off = p.offsets[f];
      const int64_t s = off[row];
      const int64_t len = row_end(off, row, p.B, p.nvalues[f]) - s;
      const int64_t* val = p.values[f] + s;
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
    if (lane == src) mine = finalize_hash(h, p.hash_mask);
  }
  if (!is_head) return;
  p.hash[idx] = mine;
  unsigned long long* tk = p.tkeys + (int64_t)g * p.C;
  uint32_t* tr = p.treps + (int64_t)g * p.C;
  const uint64_t msk = (uint64_t)p.C - 1;
  uint64_t s = (mine ^ (mine >> 29)) & msk;
  while (true) {
    const unsigned long long k = atomicCAS(&tk[s], 0ull, (unsigned long long)mine);
    if (k == 0ull || k == mine) {
      atomicMin(&tr[s], (uint32_t)i);
      p.slot_of[idx] = (uint32_t)s;
      return;
    }
    s = (s + 1) & msk;
  }
}

// ---------------------------------------------------------------- resolve
__global__ void __launch_bounds__(256) k_resolve(const __grid_constant__ DedupParams p) {
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
constexpr int NB_NT = 1024;
constexpr int NB_ITEMS = 16;

__global__ void __launch_bounds__(NB_NT) k_number(const __grid_constant__ DedupParams p) {
  const int g = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t B = p.B;
  const uint8_t* head = p.head + (int64_t)g * B;
  int32_t* cls = p.cls + (int64_t)g * B;
  int32_t* uidmap = p.uidmap + (int64_t)g * B;
  int32_t* first_rows = p.first_rows + (int64_t)g * B;
  const int fbeg = p.group_first[g], fend = p.group_first[g + 1];
  int64_t* inverse = p.inverse[g];

  __shared__ int64_t s_scan[32];
  __shared__ int64_t s_carry_len[RECD_MAX_FEAT];
  for (int f = tid; f < RECD_MAX_FEAT; f += NB_NT) s_carry_len[f] = 0;
  int64_t carry_rh = -1, carry_uid = 0;
  __syncthreads();

  constexpr int TILE = NB_NT * NB_ITEMS;
  for (int64_t tb = 0; tb < B; tb += TILE) {
    const int64_t i0 = tb + (int64_t)tid * NB_ITEMS;
    // (a) run heads: inclusive max-scan of (head ? i : -1)
    int64_t lrh = -1;
#pragma unroll
    for (int k = 0; k < NB_ITEMS; ++k) {
      const int64_t i = i0 + k;
      if (i < B && head[i]) lrh = i;
    }
    int64_t tot;
    int64_t incl = block_inclusive_max<NB_NT>(lrh, s_scan, &tot);
    // exclusive prefix = inclusive of previous thread
    int64_t prev = __shfl_up_sync(0xffffffffu, incl, 1);
    if ((tid & 31) == 0) prev = -1;
    __shared__ int64_t s_warp_last[32];
    if ((tid & 31) == 31) s_warp_last[tid >> 5] = incl;
    __syncthreads();
    if ((tid & 31) == 0 && tid > 0) prev = s_warp_last[(tid >> 5) - 1];
    int64_t rh = max(prev, carry_rh);
    // (b) class representative of every row, (c) first-occurrence flags
    int32_t cl[NB_ITEMS];
    int nfirst = 0;
#pragma unroll
    for (int k = 0; k < NB_ITEMS; ++k) {
      const int64_t i = i0 + k;
      cl[k] = -1;
      if (i < B) {
        if (head[i]) rh = i;
        cl[k] = cls[rh];
        nfirst += (cl[k] == (int32_t)i);
      }
    }
    carry_rh = max(carry_rh, tot);
    int64_t utot;
    int64_t uid = carry_uid + block_exclusive_scan<NB_NT>(nfirst, s_scan, &utot);
    // (d) uid map + first rows; (e) unique offsets per feature
#pragma unroll
    for (int k = 0; k < NB_ITEMS; ++k) {
      const int64_t i = i0 + k;
      if (i < B && cl[k] == (int32_t)i) {
        uidmap[i] = (int32_t)uid;
        first_rows[uid] = (int32_t)i;
        ++uid;
      }
    }
    for (int f = fbeg; f < fend; ++f) {
      const int64_t* off = p.offsets[f];
      const int64_t nv = p.nvalues[f];
      int64_t lsum = 0;
#pragma unroll
      for (int k = 0; k < NB_ITEMS; ++k) {
        const int64_t i = i0 + k;
        if (i < B && cl[k] == (int32_t)i) lsum += row_end(off, i, B, nv) - off[i];
      }
      int64_t ltot;
      int64_t o = s_carry_len[f] + block_exclusive_scan<NB_NT>(lsum, s_scan, &ltot);
      int64_t* uoff = p.uoffsets[f];
#pragma unroll
      for (int k = 0; k < NB_ITEMS; ++k) {
        const int64_t i = i0 + k;
        if (i < B && cl[k] == (int32_t)i) {
          uoff[uidmap[i]] = o;
          o += row_end(off, i, B, nv) - off[i];
        }
      }
      __syncthreads();
      if (tid == 0) s_carry_len[f] += ltot;
    }
    carry_uid += utot;
    __syncthreads();  // uidmap writes of this tile visible block-wide
    // (g) inverse
#pragma unroll
    for (int k = 0; k < NB_ITEMS; ++k) {
      const int64_t i = i0 + k;
      if (i < B) inverse[i] = uidmap[cl[k]];
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int f = fbeg; f < fend; ++f) {
      p.count_rows[f] = carry_uid;
      p.count_vals[f] = s_carry_len[f];
    }
  }
}

// ------------------------------------------------------------------- copy
__global__ void __launch_bounds__(256) k_copy(const __grid_constant__ DedupParams p) {
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      acc += p.count_rows[f];
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t total = s_pref[p.F];
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    int f = 0;
    while (f + 1 < p.F && s_pref[f + 1] <= w) ++f;
    const int64_t u = w - s_pref[f];
    const int g = p.feat_group[f];
    const int64_t row = p.first_rows[(int64_t)g * p.B + u];
    const int64_t* off = p.offsets[f];
    const int64_t s = off[row];
    const int64_t len = row_end(off, row, p.B, p.nvalues[f]) - s;
    const int64_t* src = p.values[f] + s;
    int64_t* dst = p.uvalues[f] + p.uoffsets[f][u];
    for (int64_t k = lane; k < len; k += 32) dst[k] = src[k];
  }
}

struct DedupScratch {
  uint8_t* head;
  uint64_t* hash;
  uint32_t* slot_of;
  int32_t *cls, *uidmap, *first_rows, *fb_list, *collide;
  unsigned long long* tkeys;
  uint32_t* treps;
};

static size_t carve_dedup(void* base, size_t cap, int G, int64_t B, int64_t C, DedupScratch* s) {
  Arena a(base, cap);
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
  (void)num_features;
  DedupScratch s;
  // groups are processed in chunks of <= RECD_MAX_FEAT features; size for all
  return carve_dedup(nullptr, 0, std::max(num_groups, 1), batch_size, table_slots(batch_size), &s);
}

extern "C" int recd_dedup(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                          const int64_t* const* values, const int64_t* const* offsets,
                          const int64_t* num_values, int64_t* const* inverse_out,
                          int64_t* const* uoffsets_out, int64_t* const* uvalues_out,
                          int64_t* counts_out, void* scratch, size_t scratch_bytes,
                          recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_groups <= 0 || batch_size <= 0 || batch_size >= (1ll << 31) || !group_sizes)
    return RECD_ERR_ARG;
  int F = 0;
  for (int g = 0; g < num_groups; ++g) {
    if (group_sizes[g] <= 0 || group_sizes[g] > RECD_MAX_FEAT) return RECD_ERR_ARG;
    F += group_sizes[g];
  }
  const int64_t B = batch_size, C = table_slots(B);
  DedupScratch s;
  if (carve_dedup(scratch, scratch_bytes, num_groups, B, C, &s) > scratch_bytes) return RECD_ERR_SCRATCH;
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
    p.tkeys = s.tkeys + (int64_t)g0 * C;
    p.treps = s.treps + (int64_t)g0 * C;

    const int64_t rows = (int64_t)p.G * B;
    {  // groups with the most values first (their blocks are the longest)
      std::vector<std::pair<int64_t, int>> order;
      for (int g = 0; g < p.G; ++g) {
        int64_t nvg = 0;
        for (int ff = p.group_first[g]; ff < p.group_first[g + 1]; ++ff) nvg += p.nvalues[ff];
        order.push_back({-nvg, g});
      }
      std::stable_sort(order.begin(), order.end());
      for (int k = 0; k < p.G; ++k) p.rs_group[k] = order[k].second;
    }
    k_rowscan<<<dim3((unsigned)ceil_div(B, RS_RPB), p.G), RS_NT, 0, stream>>>(p);
    k_insert<<<(unsigned)ceil_div((int64_t)p.G * ceil_div(B, 32) * 32, 256), 256, 0, stream>>>(p);
    k_resolve<<<(unsigned)ceil_div(rows, 256), 256, 0, stream>>>(p);
    k_fallback<<<p.G, FB_NT, 0, stream>>>(p);
    k_number<<<p.G, NB_NT, 0, stream>>>(p);
    k_copy<<<num_sms() * 4, 256, 0, stream>>>(p);
    note_launch(6);
    RECD_LAUNCH_CHECK();
    g0 = g1;
    f0 += nf;
  }
  return RECD_OK;
}
