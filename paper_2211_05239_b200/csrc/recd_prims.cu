// Segmented stable LSD radix sort + segmented exclusive scan (sm_100a).
//
// Sort: one-sweep LSD, 8-bit digits.
//   k_os_hist    block per 16K-element chunk: digit histograms of EVERY pass
//                at once (keys read once), added to per-(segment, pass) global
//                counts; also clears the tile status words of the first pass.
//   k_os_setup   one block: per segment, tile prefix (actual counts) and the
//                exclusive digit scans -> each digit's segment-relative base.
//   k_onesweep   per pass, persistent blocks take 4096-element tiles in order
//                (atomic ticket), rank them stably (warp match_any + per-warp
//                digit counters), publish the tile's digit counts and look back
//                over the preceding tiles of the segment (decoupled look-back,
//                one thread per digit) for the tile's global digit offsets,
//                then scatter through shared memory so runs of equal digits
//                are written contiguously.  Keys and values move once per pass.
// Element order inside a tile is (warp, round, lane) == input order and tiles
// are ranked in segment order, so every pass is stable and the result
// deterministic.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "recd_prims.cuh"

namespace recd {

constexpr int OS_NT = 256;                     // threads == digits
#ifndef RECD_OS_ITEMS
#define RECD_OS_ITEMS 16
#endif
constexpr int OS_ITEMS = RECD_OS_ITEMS;
constexpr int OS_TILE = OS_NT * OS_ITEMS;      // 4096 elements per tile
constexpr int OS_WARPS = OS_NT / 32;
constexpr int OS_HCHUNK = OS_TILE * 4;         // elements per histogram block
constexpr int OS_MAXSEG = 64;
constexpr int OS_MAXPASS = 4;
constexpr uint32_t OS_AGG = 1u << 30, OS_PRE = 2u << 30, OS_CNT = (1u << 30) - 1;
#ifndef RECD_OS_LB
#define RECD_OS_LB 8
#endif
constexpr int OS_LB = RECD_OS_LB;
#ifndef RECD_OS_SETUP_CLEAR  // k_os_setup clears the sort state (no memset nodes)
#define RECD_OS_SETUP_CLEAR 1
#endif
#ifndef RECD_OS_EARLY  // publish a tile's digit counts before its ranking
#define RECD_OS_EARLY 1
#endif
#ifndef RECD_OS_LOCAL  // one-CTA-per-segment sort when every segment fits a tile
#define RECD_OS_LOCAL 1
#endif              // look-back tiles per round trip

struct OsSeg {
  int64_t base;          // element offset of the segment
  const int64_t* count;  // device: actual element count
  int64_t tcap0;         // first capacity tile (status rows)
  int64_t hchunk0;       // first histogram chunk
};

struct OsParams {
  int S, npass, pass, shift, nbits, bits;
  int64_t total_hchunks;
  int64_t total_tcap;
  OsSeg seg[OS_MAXSEG];
  const uint32_t* kin;
  const uint32_t* vin;
  uint32_t* kout;
  uint32_t* vout;
  uint32_t* ghist;     // [S][OS_MAXPASS][256]: counts, then segment-relative digit bases
  int64_t* tile0;      // [S + 1] prefix of actual tiles
  uint32_t* counters;  // [OS_MAXPASS] tile tickets
  uint32_t* status;    // [2][total_tcap][256]
  uint32_t* tmap;      // [total_tcap] ticket -> (segment << 24) | tile (RECD_OS_IL)
  int il;              // tickets interleaved over the segments (RECD_OS_IL and S > 1)
  int clear_state;     // k_os_setup zeroes the ticket counters and pass 0's status rows
  const int32_t* gate; // nullable: run only if *gate != 0
};

__device__ __forceinline__ bool os_gated_off(const OsParams& p) {
  return p.gate && *(volatile const int32_t*)p.gate == 0;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(OS_NT) k_os_hist(const __grid_constant__ OsParams p) {
  RECD_PDL_PROLOGUE();
  if (os_gated_off(p)) return;
  const int64_t chunk = blockIdx.x;
  int s = 0;
  while (s + 1 < p.S && p.seg[s + 1].hchunk0 <= chunk) ++s;
  const OsSeg& sg = p.seg[s];
  if (chunk == 0 && threadIdx.x < OS_MAXPASS) p.counters[threadIdx.x] = 0;
  const int64_t n = *sg.count;
  const int64_t lo = (chunk - sg.hchunk0) * OS_HCHUNK;
  if (lo >= n) return;
  const int64_t hi = min(n, lo + (int64_t)OS_HCHUNK);
  {  // clear the pass-0 status rows of the tiles in this chunk
    const int64_t t0 = sg.tcap0 + lo / OS_TILE, t1 = sg.tcap0 + ceil_div(hi, OS_TILE);
    for (int64_t e = t0 * 256 + threadIdx.x; e < t1 * 256; e += OS_NT) p.status[e] = 0u;
  }
  __shared__ uint32_t sh[OS_MAXPASS][256];
  for (int q = 0; q < p.npass; ++q) sh[q][threadIdx.x] = 0;
  __syncthreads();
  const uint32_t* k = p.kin + sg.base;
  constexpr int U = 8;
  for (int64_t j0 = lo; j0 < hi; j0 += OS_NT * U) {
    uint32_t kk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * OS_NT + threadIdx.x;
      kk[u] = j < hi ? __ldg(k + j) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * OS_NT + threadIdx.x;
      if (j < hi)
        for (int q = 0; q < p.npass; ++q)
          atomicAdd(&sh[q][(kk[u] >> (8 * q)) & ((1u << min(8, p.bits - 8 * q)) - 1u)], 1u);
    }
  }
  __syncthreads();
  for (int q = 0; q < p.npass; ++q) {
    const uint32_t c = sh[q][threadIdx.x];
    if (c) atomicAdd(&p.ghist[((int64_t)s * OS_MAXPASS + q) * 256 + threadIdx.x], c);
  }
}

// Tile order (RECD_OS_IL): a pass's persistent CTAs take tiles by ticket, and
// a tile's global digit offsets come from the decoupled look-back: it sums
// the aggregates of the tiles before it in its segment back to the nearest
// published inclusive prefix, OS_LB tiles per L2 round trip.  In
// segment-major ticket order the ~440 tiles in flight sit in one or two
// segments, so a tile walks back over many in-flight predecessors;
// interleaving the tickets over the segments in proportion to their sizes
// (tile j of segment s at fraction (j + 1) / T_s of the pass) leaves ~17 per
// segment.  Results are identical: a tile's offsets are integer sums over its
// own segment's predecessors, which still take earlier tickets.  A/B (with
// early publication): occurrence stage 0.715-0.719 vs 0.770-0.776 ms.
#ifndef RECD_OS_IL
#define RECD_OS_IL 1
#endif
// ticket of tile j of segment s: its rank in (j + 1) / T_s, ties to the lower
// segment (integer arithmetic, so the map is a permutation)
__device__ __forceinline__ int64_t il_ticket(const int64_t* T, int S, int s, int64_t j) {
  int64_t t = j;
  const int64_t Ts = T[s];
  for (int s2 = 0; s2 < S; ++s2) {
    if (s2 == s || T[s2] == 0) continue;
    const int64_t X = (j + 1) * T[s2];
    int64_t c = (X - 1) / Ts;            // tiles j' of s2 with (j' + 1) / T_s2 < (j + 1) / T_s
    if (s2 < s && X % Ts == 0) ++c;      // ... and the tie
    t += min(c, T[s2]);
  }
  return t;
}

// block per (segment, pass): exclusive digit scan; block 0 also the tile
// prefix; every block a slice of the interleaved ticket map
__global__ void __launch_bounds__(OS_NT) k_os_setup(const __grid_constant__ OsParams p) {
  RECD_PDL_PROLOGUE();
  if (os_gated_off(p)) return;
  __shared__ int64_t s_scan[32];
  if (p.clear_state) {  // (instead of two memset nodes before this kernel)
    if (blockIdx.x == 0 && threadIdx.x < OS_MAXPASS) p.counters[threadIdx.x] = 0u;
    const int64_t words = p.total_tcap * 256;
    uint2* st2 = reinterpret_cast<uint2*>(p.status);  // 8-byte aligned (counters + 64 words)
    for (int64_t i = (int64_t)blockIdx.x * OS_NT + threadIdx.x; i < words / 2; i += (int64_t)gridDim.x * OS_NT)
      st2[i] = make_uint2(0u, 0u);
  }
  if (p.il) {
    __shared__ int64_t s_T[OS_MAXSEG], s_p[OS_MAXSEG + 1];
    for (int q = threadIdx.x; q < p.S; q += OS_NT) s_T[q] = ceil_div(*p.seg[q].count, (int64_t)OS_TILE);
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int q = 0; q < p.S; ++q) s_p[q] = t, t += s_T[q];
      s_p[p.S] = t;
    }
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * OS_NT + threadIdx.x; i < s_p[p.S]; i += (int64_t)gridDim.x * OS_NT) {
      int s = 0, hi = p.S - 1;
      while (s < hi) {
        const int mid = (s + hi + 1) >> 1;
        if (s_p[mid] <= i) s = mid; else hi = mid - 1;
      }
      const int64_t j = i - s_p[s];
      p.tmap[il_ticket(s_T, p.S, s, j)] = ((uint32_t)s << 24) | (uint32_t)j;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t t = 0;
    for (int s = 0; s < p.S; ++s) {
      p.tile0[s] = t;
      t += ceil_div(*p.seg[s].count, OS_TILE);
    }
    p.tile0[p.S] = t;
  }
  const int s = blockIdx.x / p.npass, q = blockIdx.x - s * p.npass;
  uint32_t* h = p.ghist + ((int64_t)s * OS_MAXPASS + q) * 256;
  const uint32_t c = h[threadIdx.x];
  int64_t tot;
  const int64_t x = block_exclusive_scan<OS_NT>(c, s_scan, &tot);
  h[threadIdx.x] = (uint32_t)x;
}

// decoupled look-back, OS_LB predecessors per round trip: the loads of tiles
// k, k-1, ..., k-OS_LB+1 are independent, so a walk over many in-flight tiles
// costs one L2 latency per OS_LB tiles instead of per tile; the words are
// consumed in order up to the first unpublished one (retried) or the first
// inclusive prefix (done); tile 0 always publishes a prefix.  col = this
// thread's digit column of the segment's status rows; returns the exclusive
// count of tile lt_ (> 0).
__device__ __forceinline__ uint32_t os_look_back(const uint32_t* col, int64_t lt_) {
  uint32_t excl = 0;
  for (int64_t k = lt_ - 1;;) {
    uint32_t v[OS_LB];
#pragma unroll
    for (int j = 0; j < OS_LB; ++j) v[j] = (k - j >= 0) ? ld_relaxed(col + (k - j) * 256) : OS_PRE;
    int j = 0;
    bool done = false;
#pragma unroll
    for (int q = 0; q < OS_LB; ++q) {
      if (done || j < q) continue;                  // stopped earlier in this batch
      const uint32_t w = v[q];
      if ((w & ~OS_CNT) == 0u) continue;            // not published yet: retry from here
      excl += w & OS_CNT;
      if (w & OS_PRE) done = true;
      j = q + 1;
    }
    if (done) break;
    k -= j;
  }
  return excl;
}

#ifndef RECD_OS_MINB
#define RECD_OS_MINB 3
#endif
__global__ void __launch_bounds__(OS_NT, RECD_OS_MINB) k_onesweep(const __grid_constant__ OsParams p) {
  RECD_PDL_PROLOGUE();
  if (os_gated_off(p)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t mask = (1u << p.nbits) - 1u;
  const unsigned lt = lanemask_lt();
  __shared__ uint32_t s_wcnt[OS_WARPS][256];
  __shared__ uint32_t s_tdb[256];
  __shared__ uint32_t s_gb[256];
  __shared__ uint32_t s_keys[OS_TILE];
  __shared__ uint32_t s_vals[OS_TILE];
  __shared__ int64_t s_scan[32];
  __shared__ int64_t s_tile;
  __shared__ int64_t s_t0[OS_MAXSEG + 1];
  for (int q = tid; q <= p.S; q += OS_NT) s_t0[q] = p.tile0[q];
  uint32_t* st_cur = p.status + (int64_t)(p.pass & 1) * p.total_tcap * 256;
  uint32_t* st_next = p.status + (int64_t)((p.pass + 1) & 1) * p.total_tcap * 256;
  __syncthreads();
  const int64_t total = s_t0[p.S];
  while (true) {
    if (tid == 0) s_tile = atomicAdd(&p.counters[p.pass], 1u);
    __syncthreads();
    const int64_t t = s_tile;
    if (t >= total) break;
    int s = 0;
    int64_t lt_;
    if (p.il) {
      const uint32_t m = __ldg(p.tmap + t);
      s = (int)(m >> 24);
      lt_ = (int64_t)(m & 0xffffffu);
    } else {
      int shi = p.S - 1;  // last segment whose first tile <= t
      while (s < shi) {
        const int mid = (s + shi + 1) >> 1;
        if (s_t0[mid] <= t) s = mid; else shi = mid - 1;
      }
      lt_ = t - s_t0[s];
    }
    const OsSeg& sg = p.seg[s];
    const int64_t n = *sg.count;
    const int64_t lo = lt_ * OS_TILE;
    const int tn = (int)min((int64_t)OS_TILE, n - lo);
    const uint32_t* kin = p.kin + sg.base + lo;
    const uint32_t* vin = p.vin + sg.base + lo;
    for (int d = lane; d < 256; d += 32) s_wcnt[warp][d] = 0;
    __syncwarp();
    uint32_t key[OS_ITEMS], val[OS_ITEMS], rank[OS_ITEMS];
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {
      const int e = warp * (OS_TILE / OS_WARPS) + r * 32 + lane;
      key[r] = e < tn ? __ldg(kin + e) : 0u;
      val[r] = e < tn ? __ldg(vin + e) : 0u;
    }
    uint32_t* my = st_cur + (sg.tcap0 + lt_) * 256 + tid;
#if RECD_OS_EARLY
    // publish the tile's digit counts before ranking it (shared-atomic
    // histogram): the tiles behind it in the look-back stop waiting for this
    // tile's ranking (ncu: 27% of a pass's stall samples sat in the look-back)
    s_tdb[tid] = 0u;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {
      const int e = warp * (OS_TILE / OS_WARPS) + r * 32 + lane;
      if (e < tn) atomicAdd(&s_tdb[(key[r] >> p.shift) & mask], 1u);
    }
    __syncthreads();
    st_relaxed(my, (lt_ == 0 ? OS_PRE : OS_AGG) | s_tdb[tid]);
#endif
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {
      const int e = warp * (OS_TILE / OS_WARPS) + r * 32 + lane;
      const bool valid = e < tn;
      const uint32_t d = valid ? ((key[r] >> p.shift) & mask) : 0x100u;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      uint32_t before = 0;
      if (valid) before = s_wcnt[warp][d];
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) s_wcnt[warp][d] = before + __popc(peers);
      __syncwarp();
      rank[r] = before + __popc(peers & lt);
    }
    __syncthreads();
    // thread tid owns digit tid: per-warp bases, tile count, publish, look back
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < OS_WARPS; ++w) {
      const uint32_t c = s_wcnt[w][tid];
      s_wcnt[w][tid] = cnt;
      cnt += c;
    }
    uint32_t excl = 0;
    if (lt_ == 0) {
      if (!RECD_OS_EARLY) st_relaxed(my, OS_PRE | cnt);
    } else {
      if (!RECD_OS_EARLY) st_relaxed(my, OS_AGG | cnt);
      excl = os_look_back(st_cur + sg.tcap0 * 256 + tid, lt_);
      st_relaxed(my, OS_PRE | (excl + cnt));
    }
    if (p.pass + 1 < p.npass) st_next[(sg.tcap0 + lt_) * 256 + tid] = 0u;
    s_gb[tid] = (uint32_t)(sg.base + p.ghist[((int64_t)s * OS_MAXPASS + p.pass) * 256 + tid] + excl);
    int64_t tot;
    const int64_t tdb = block_exclusive_scan<OS_NT>(cnt, s_scan, &tot);
    s_tdb[tid] = (uint32_t)tdb;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {
      const int e = warp * (OS_TILE / OS_WARPS) + r * 32 + lane;
      if (e < tn) {
        const uint32_t d = (key[r] >> p.shift) & mask;
        const uint32_t lp = s_tdb[d] + s_wcnt[warp][d] + rank[r];
        s_keys[lp] = key[r];
        s_vals[lp] = val[r];
      }
    }
    __syncthreads();
    for (int q = tid; q < tn; q += OS_NT) {
      const uint32_t k = s_keys[q];
      const uint32_t d = (k >> p.shift) & mask;
      const uint32_t pos = s_gb[d] + (uint32_t)q - s_tdb[d];
      p.kout[pos] = k;
      p.vout[pos] = s_vals[q];
    }
    __syncthreads();
  }
}

// Small sorts (every segment fits one tile, e.g. config 1's inverse CSR: 8
// segments of 4,096 rows): one CTA per segment runs every pass in shared
// memory -- same stable warp ranking as k_onesweep, no histogram pass, no
// look-back, no global round trip between passes, one launch instead of
// memset + k_os_hist + k_os_setup + one k_onesweep per pass.  The result goes
// where the multi-pass sort would leave it (alt buffers for an odd pass count).
__global__ void __launch_bounds__(LS_NT) k_local_sort(const __grid_constant__ OsParams p) {
  RECD_PDL_PROLOGUE();
  if (os_gated_off(p)) return;
  __shared__ LocalSortSmem sm;
  const OsSeg& sg = p.seg[blockIdx.x];
  const int tn = (int)min((int64_t)LS_TILE, *sg.count);
  uint32_t key[LS_ITEMS], val[LS_ITEMS];
#pragma unroll
  for (int r = 0; r < LS_ITEMS; ++r) {
    const int e = ls_elem(r);
    key[r] = e < tn ? __ldg(p.kin + sg.base + e) : 0u;
    val[r] = e < tn ? __ldg(p.vin + sg.base + e) : 0u;
  }
  local_sort_tile(key, val, tn, p.bits, sm);
  uint32_t* ko = (p.npass & 1) ? p.kout : const_cast<uint32_t*>(p.kin);
  uint32_t* vo = (p.npass & 1) ? p.vout : const_cast<uint32_t*>(p.vin);
  for (int e = threadIdx.x; e < tn; e += LS_NT) {
    ko[sg.base + e] = sm.keys[e];
    vo[sg.base + e] = sm.vals[e];
  }
}

static void build_os_params(const SegDesc* segs, int S, OsParams* p) {
  memset(p, 0, sizeof(*p));
  p->S = S;
  int64_t tc = 0, hc = 0;
  for (int s = 0; s < S; ++s) {
    p->seg[s].base = segs[s].base;
    p->seg[s].count = segs[s].count;
    p->seg[s].tcap0 = tc;
    p->seg[s].hchunk0 = hc;
    tc += std::max<int64_t>(1, ceil_div(segs[s].cap, OS_TILE));
    hc += std::max<int64_t>(1, ceil_div(segs[s].cap, OS_HCHUNK));
  }
  p->total_tcap = tc;
  p->total_hchunks = hc;
}

// scratch words: ghist + tile0 (int64) + counters + 2 status planes + ticket map
static int64_t os_words(const OsParams& p) {
  return (int64_t)OS_MAXSEG * OS_MAXPASS * 256 + 2 * (OS_MAXSEG + 1) + 64 + 2 * p.total_tcap * 256 +
         p.total_tcap;
}

int64_t sort_hist_words(const SegDesc* segs, int S) {
  int64_t words = 0;
  for (int s0 = 0; s0 < S; s0 += OS_MAXSEG) {
    OsParams p;
    build_os_params(segs + s0, std::min(OS_MAXSEG, S - s0), &p);
    words = std::max(words, os_words(p));
  }
  return words;
}

// persistent sort CTAs per SM (RECD_OS_CTAS env: fewer than the occupancy
// limit leaves SM slots to a kernel running beside the sort on another stream)
static int os_grid() {
  static int g = 0;
  if (!g) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_onesweep, OS_NT, 0);
    per = std::max(per, 1);
    if (const char* e = getenv("RECD_OS_CTAS")) per = std::max(1, std::min(per, atoi(e)));
    g = num_sms() * per;
  }
  return g;
}

int seg_sort_pairs(const SegDesc* segs, int S, int bits, uint32_t* keys, uint32_t* vals,
                   uint32_t* keys_alt, uint32_t* vals_alt, uint32_t* hist, bool* in_alt,
                   cudaStream_t stream, const int32_t* gate, bool hist_ready) {
  *in_alt = false;
  if (S <= 0 || bits <= 0) return RECD_OK;
  const int npass = (bits + 7) / 8;
  if (npass > OS_MAXPASS) return RECD_ERR_UNSUPPORTED;
  for (int s = 0; s < S; ++s)
    if (segs[s].cap > (int64_t)OS_CNT) return RECD_ERR_UNSUPPORTED;
  bool local = RECD_OS_LOCAL != 0;
  for (int s = 0; s < S; ++s) local &= segs[s].cap <= LS_TILE;
  for (int s0 = 0; s0 < S; s0 += OS_MAXSEG) {
    OsParams p;
    build_os_params(segs + s0, std::min(OS_MAXSEG, S - s0), &p);
    p.npass = npass;
    if (local) {
      p.bits = bits;
      p.gate = gate;
      p.kin = keys; p.vin = vals; p.kout = keys_alt; p.vout = vals_alt;
      pdl(k_local_sort, p.S, LS_NT, 0, stream)(p);
      note_launch();
      continue;
    }
    p.bits = bits;
    p.gate = gate;
    p.ghist = hist;
    p.tile0 = reinterpret_cast<int64_t*>(hist + (int64_t)OS_MAXSEG * OS_MAXPASS * 256);
    p.counters = reinterpret_cast<uint32_t*>(p.tile0 + OS_MAXSEG + 1);
    p.status = p.counters + 64;
    p.tmap = p.status + 2 * p.total_tcap * 256;
    // (sorts of short segments -- the inverse CSR: 16 tiles each at cfg2 --
    // gain nothing and would pay the map's setup on the critical path)
    p.il = RECD_OS_IL && p.S > 1 && p.total_tcap >= 64 * (int64_t)p.S;
    p.kin = keys;
    if (hist_ready && S <= OS_MAXSEG) {
      // the producer of the keys already counted every pass's digits into
      // ghist (sort_hist_clear + its own smem histograms): only the ticket
      // counters and the first pass's tile status words need clearing
      if (RECD_OS_SETUP_CLEAR) {
        p.clear_state = 1;
      } else {
        RECD_CUDA_CHECK(cudaMemsetAsync(p.counters, 0, sizeof(uint32_t) * OS_MAXPASS, stream));
        RECD_CUDA_CHECK(cudaMemsetAsync(p.status, 0, sizeof(uint32_t) * p.total_tcap * 256, stream));
      }
      pdl(k_os_setup, p.S * npass, OS_NT, 0, stream)(p);
      note_launch(1);
    } else {
      RECD_CUDA_CHECK(cudaMemsetAsync(p.ghist, 0, sizeof(uint32_t) * p.S * OS_MAXPASS * 256, stream));
      pdl(k_os_hist, (unsigned)p.total_hchunks, OS_NT, 0, stream)(p);
      pdl(k_os_setup, p.S * npass, OS_NT, 0, stream)(p);
      note_launch(2);
    }
    uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
    for (int pass = 0; pass < npass; ++pass) {
      p.pass = pass;
      p.shift = 8 * pass;
      p.nbits = std::min(8, bits - 8 * pass);
      p.kin = ki; p.vin = vi; p.kout = ko; p.vout = vo;
      pdl(k_onesweep, (unsigned)std::min<int64_t>(os_grid(), p.total_tcap), OS_NT, 0, stream)(p);
      note_launch();
      std::swap(ki, ko);
      std::swap(vi, vo);
    }
  }
  *in_alt = (npass % 2) == 1;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

int sort_hist_clear(int S, uint32_t* hist, cudaStream_t stream) {
  RECD_CUDA_CHECK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * std::min(S, OS_MAXSEG) * OS_MAXPASS * 256,
                                  stream));
  return RECD_OK;
}

// ------------------------------------------------------------------- scan
constexpr int XS_NT = 256;
constexpr int XS_ITEMS = 16;
constexpr int XS_CHUNK = XS_NT * XS_ITEMS;  // 4096
constexpr int XS_MAXSEG = 48;

struct ScanSegDev {
  const int64_t* in;
  int64_t* out;
  int64_t cap;
  const int64_t* count;
  int64_t* total;
  int64_t chunk0;
  int64_t nchunks;
};
struct ScanParams {
  int S;
  int64_t total_chunks;
  ScanSegDev seg[XS_MAXSEG];
  int64_t* part;
};

__device__ __forceinline__ int scan_seg(const ScanParams& p, int64_t chunk) {
  int lo = 0, hi = p.S - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.seg[mid].chunk0 <= chunk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(XS_NT) k_scan_reduce(const __grid_constant__ ScanParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t chunk = blockIdx.x;
  const ScanSegDev& sg = p.seg[scan_seg(p, chunk)];
  const int64_t n = sg.count ? *sg.count : sg.cap;
  const int64_t lo = (chunk - sg.chunk0) * XS_CHUNK;
  int64_t sum = 0;
  for (int64_t j = lo + threadIdx.x; j < min(n, lo + (int64_t)XS_CHUNK); j += XS_NT) sum += sg.in[j];
  __shared__ int64_t s_scan[32];
  int64_t tot;
  block_exclusive_scan<XS_NT>(sum, s_scan, &tot);
  if (threadIdx.x == 0) p.part[chunk] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_parts(const __grid_constant__ ScanParams p) {
  RECD_PDL_PROLOGUE();
  const ScanSegDev& sg = p.seg[blockIdx.x];
  __shared__ int64_t s_scan[32];
  int64_t carry = 0;
  for (int64_t tb = 0; tb < sg.nchunks; tb += 1024) {
    const int64_t c = tb + threadIdx.x;
    const int64_t v = c < sg.nchunks ? p.part[sg.chunk0 + c] : 0;
    int64_t tot;
    const int64_t x = block_exclusive_scan<1024>(v, s_scan, &tot);
    if (c < sg.nchunks) p.part[sg.chunk0 + c] = carry + x;
    carry += tot;
  }
  if (threadIdx.x == 0 && sg.total) *sg.total = carry;
}

__global__ void __launch_bounds__(XS_NT) k_scan_down(const __grid_constant__ ScanParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t chunk = blockIdx.x;
  const ScanSegDev& sg = p.seg[scan_seg(p, chunk)];
  const int64_t n = sg.count ? *sg.count : sg.cap;
  const int64_t lo = (chunk - sg.chunk0) * XS_CHUNK;
  if (lo >= n) return;
  const int64_t j0 = lo + (int64_t)threadIdx.x * XS_ITEMS;
  int64_t v[XS_ITEMS];
  int64_t sum = 0;
#pragma unroll
  for (int t = 0; t < XS_ITEMS; ++t) {
    v[t] = (j0 + t < n) ? sg.in[j0 + t] : 0;
    sum += v[t];
  }
  __shared__ int64_t s_scan[32];
  int64_t tot;
  int64_t x = p.part[chunk] + block_exclusive_scan<XS_NT>(sum, s_scan, &tot);
#pragma unroll
  for (int t = 0; t < XS_ITEMS; ++t) {
    if (j0 + t < n) sg.out[j0 + t] = x;
    x += v[t];
  }
}

static void build_scan_params(const ScanDesc* segs, int S, ScanParams* p) {
  memset(p, 0, sizeof(*p));
  p->S = S;
  int64_t chunk = 0;
  for (int s = 0; s < S; ++s) {
    p->seg[s].in = segs[s].in;
    p->seg[s].out = segs[s].out;
    p->seg[s].cap = segs[s].cap;
    p->seg[s].count = segs[s].count;
    p->seg[s].total = segs[s].total;
    p->seg[s].chunk0 = chunk;
    p->seg[s].nchunks = std::max<int64_t>(1, ceil_div(segs[s].cap, XS_CHUNK));
    chunk += p->seg[s].nchunks;
  }
  p->total_chunks = chunk;
}

int64_t scan_part_words(const ScanDesc* segs, int S) {
  int64_t words = 0;
  for (int s0 = 0; s0 < S; s0 += XS_MAXSEG) {
    ScanParams p;
    build_scan_params(segs + s0, std::min(XS_MAXSEG, S - s0), &p);
    words = std::max(words, p.total_chunks);
  }
  return words;
}

int seg_exclusive_scan(const ScanDesc* segs, int S, int64_t* part, cudaStream_t stream) {
  for (int s0 = 0; s0 < S; s0 += XS_MAXSEG) {
    ScanParams p;
    build_scan_params(segs + s0, std::min(XS_MAXSEG, S - s0), &p);
    p.part = part;
    pdl(k_scan_reduce, (unsigned)p.total_chunks, XS_NT, 0, stream)(p);
    pdl(k_scan_parts, p.S, 1024, 0, stream)(p);
    pdl(k_scan_down, (unsigned)p.total_chunks, XS_NT, 0, stream)(p);
    note_launch(3);
  }
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

}  // namespace recd

using namespace recd;

// Segmented stable radix sort of (uint32 key, uint32 value) pairs by the low
// `bits` bits of the key (the primitive under the backward's inverse CSR and
// occurrence sort; exported for tests and reuse).  Segment s occupies
// [bases[s], bases[s] + caps[s]) of keys/vals, *device_counts[s] elements
// valid; the result is left in keys/vals (*in_alt_out = 0) or keys_alt/vals_alt
// (*in_alt_out = 1).
extern "C" size_t recd_sort_pairs_scratch_bytes(int32_t num_segments, const int64_t* bases,
                                                const int64_t* caps) {
  std::vector<SegDesc> segs;
  for (int s = 0; s < num_segments; ++s) segs.push_back({bases[s], caps[s], nullptr});
  return (size_t)std::max<int64_t>(sort_hist_words(segs.data(), num_segments), 256) * sizeof(uint32_t);
}

extern "C" int recd_sort_pairs(int32_t num_segments, const int64_t* bases, const int64_t* caps,
                               const int64_t* const* device_counts, int32_t bits, uint32_t* keys,
                               uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                               int32_t* in_alt_out, void* scratch, size_t scratch_bytes,
                               recd_stream_t stream) {
  if (num_segments <= 0 || bits < 0 || bits > 32 || !device_counts || !in_alt_out) return RECD_ERR_ARG;
  if (recd_sort_pairs_scratch_bytes(num_segments, bases, caps) > scratch_bytes) return RECD_ERR_SCRATCH;
  std::vector<SegDesc> segs;
  for (int s = 0; s < num_segments; ++s) segs.push_back({bases[s], caps[s], device_counts[s]});
  bool alt = false;
  const int rc = seg_sort_pairs(segs.data(), num_segments, bits, keys, vals, keys_alt, vals_alt,
                                reinterpret_cast<uint32_t*>(scratch), &alt, (cudaStream_t)stream);
  *in_alt_out = alt ? 1 : 0;
  return rc;
}
