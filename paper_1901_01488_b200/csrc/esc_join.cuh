// esc_join.cuh — hash joins over the device-resident ESC temps, included
// by esc_kernels.cu.
//
//   esc_hash_insert   HashTableIndex._insert_all   (executor.py:304-325)
//   esc_hash_probe    HashTableIndex.probe_groups  (executor.py:327-346)
//   esc_expand        _expand_matches + np.repeat  (executor.py:373-386, :436-447)
//   esc_join_count    the fused probe pipeline of a COUNT(*) plan (executor.py:403-474): one
//                     pass over the probe table's key columns, every hash lookup and the
//                     per-stage tuple counts fused, nothing expanded.
//
// The table is the reference's: open addressing, splitmix64 of the key's 64-bit pattern, linear
// probing, capacity a power of two at load <= 0.7, slots hold dense group ids (= index into the
// ascending unique keys).  Inserting with atomicCAS instead of the reference's sorted rounds puts
// keys in different slots of a probe run, but every lookup returns the same group id, so groups,
// counts, row sets and row order are identical.
//
// esc_join_count: a COUNT over a join tree never needs the expanded tuples.  The host folds every
// step into a per-group weight (group size x the weights of the steps probed from its rows,
// computed bottom-up per stage prefix), so a probe row contributes prod_t weight_t[group_t(row)]
// to each stage.  For a star (every probe key on the probe table) the weights are stage-invariant
// and are handed over as dense "factor" arrays indexed by key - min: 1-bit for primary-key
// dimensions.  Small factor arrays are staged in shared memory, so the pass streams the probe
// table's key columns at HBM speed with all lookups on-chip.
#pragma once

namespace esc {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void hash_insert_kernel(const long long* __restrict__ uk, int64_t n, unsigned long long* slots,
                                   unsigned long long mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long pos = splitmix64((unsigned long long)uk[i]) & mask;
    while (atomicCAS(&slots[pos], ~0ull, (unsigned long long)i) != ~0ull) pos = (pos + 1) & mask;
  }
}

// occ: the table's occupancy bits (staged in shared memory) or nullptr.  A key whose home slot is
// empty is absent (linear probing), so at load <= 1/4 about three quarters of the non-members
// are rejected on chip, without the dependent L2 load
__device__ __forceinline__ unsigned long long pairs_find(const longlong2* __restrict__ pairs, unsigned long long mask,
                                                         long long k, const uint32_t* occ) {
  unsigned long long h = splitmix64((unsigned long long)k) & mask;
  if (occ != nullptr && !((occ[h >> 5] >> (h & 31)) & 1u)) return 0;
  for (;;) {
    const longlong2 e = __ldg(pairs + h);
    if (e.y == 0) return 0;
    if (e.x == k) return (unsigned long long)e.y;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ long long hash_find(const long long* __restrict__ slots, unsigned long long mask,
                                               const long long* __restrict__ uk, long long key) {
  unsigned long long pos = splitmix64((unsigned long long)key) & mask;
  while (true) {
    const long long s = __ldg(slots + pos);
    if (s < 0) return -1;
    if (__ldg(uk + s) == key) return s;
    pos = (pos + 1) & mask;
  }
}

__device__ __forceinline__ long long ld_key(const uint8_t* base, int dtype, int64_t row) {
  switch (dtype) {
    case ESC_I8: return reinterpret_cast<const int8_t*>(base)[row];
    case ESC_I16: return reinterpret_cast<const int16_t*>(base)[row];
    case ESC_I32: return reinterpret_cast<const int32_t*>(base)[row];
    case ESC_U8: return reinterpret_cast<const uint8_t*>(base)[row];
    case ESC_U16: return reinterpret_cast<const uint16_t*>(base)[row];
    case ESC_U32: return reinterpret_cast<const uint32_t*>(base)[row];
    default: return reinterpret_cast<const long long*>(base)[row];
  }
}

struct ProbeParams {
  const long long* slots;
  unsigned long long mask;
  const long long* uk;
  const uint8_t* keys;
  int32_t dtype;
  const uint8_t* nulls;
  const int64_t* rows;
  const uint8_t* valid;
  int64_t n;
  long long* out;
};

__global__ void hash_probe_kernel(const ProbeParams p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
    long long g = -1;
    const int64_t r = p.rows ? p.rows[i] : i;
    if ((p.valid == nullptr || p.valid[i]) && (p.nulls == nullptr || p.nulls[r] == 0))
      g = hash_find(p.slots, p.mask, p.uk, ld_key(p.keys, p.dtype, r));
    p.out[i] = g;
  }
}

// one thread per tuple: its matches, in group order, at its exclusive offset
__global__ void expand_kernel(const long long* __restrict__ groups, const long long* __restrict__ offsets, int64_t n,
                              const long long* __restrict__ gstart, const long long* __restrict__ grows,
                              long long* __restrict__ out_tuple, long long* __restrict__ out_row) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long g = groups[i];
    if (g < 0) continue;
    const long long s = gstart[g], e = gstart[g + 1];
    long long o = offsets[i];
    for (long long j = s; j < e; ++j, ++o) {
      if (out_tuple) out_tuple[o] = i;
      out_row[o] = grows[j];
    }
  }
}

// ---- fused COUNT probe ------------------------------------------------------------------------
struct JoinStepK {
  const uint8_t* keys;
  const uint8_t* nulls;
  int32_t dtype;
  int32_t mode;         // ESC_JOIN_DENSE / ESC_JOIN_HASH
  long long dmin;
  long long dlen;
  const uint8_t* factor;  // global factor array (dense)
  int32_t fbits;          // 1, 8, 16, 32, 64
  uint32_t smem_off;      // byte offset of the staged factor array, or kNoSmem
  const long long* slots;
  unsigned long long mask;
  const long long* uk;
  const unsigned long long* weight[ESC_MAX_STEPS + 1];
  const uint32_t* occ;    // PAIRS: the table's occupancy bits (capacity / 32 words after the pairs)
};

constexpr uint32_t kNoSmem = 0xFFFFFFFFu;

struct JoinParams {
  int32_t n_steps;
  int32_t n_stages;
  int32_t star;
  int32_t bits;  // semi-join star: 1-bit dense factors, int32 keys without NULLs -> join_bits_kernel
  int64_t nrows;
  const uint32_t* bitmap;
  int32_t stage_of[ESC_MAX_STEPS];
  JoinStepK steps[ESC_MAX_STEPS];
  uint32_t smem_bytes;
  unsigned long long* out;  // [n_stages + 1]
};

__device__ __forceinline__ unsigned long long factor_at(const uint8_t* f, int bits, long long i) {
  switch (bits) {
    case 1: return (reinterpret_cast<const uint32_t*>(f)[i >> 5] >> (i & 31)) & 1u;
    case 8: return f[i];
    case 16: return reinterpret_cast<const uint16_t*>(f)[i];
    case 32: return reinterpret_cast<const uint32_t*>(f)[i];
    default: return reinterpret_cast<const unsigned long long*>(f)[i];
  }
}

constexpr int kJoinThreads = 512;

__global__ void __launch_bounds__(kJoinThreads, 2) join_count_kernel(const __grid_constant__ JoinParams p) {
  extern __shared__ __align__(16) uint8_t jsm[];
  // stage the small dense factor arrays (all lookups of the pass then stay on chip)
  for (int t = 0; t < p.n_steps; ++t) {
    const JoinStepK& s = p.steps[t];
    if (s.smem_off == kNoSmem) continue;
    const bool pairs = s.mode == ESC_JOIN_PAIRS;
    const long long bytes = pairs ? (long long)((s.mask + 1) / 8)
                                  : s.fbits == 1 ? ((s.dlen + 31) / 32) * 4 : s.dlen * (s.fbits / 8);
    const long long words = (bytes + 15) / 16;
    const uint4* src = reinterpret_cast<const uint4*>(pairs ? reinterpret_cast<const uint8_t*>(s.occ) : s.factor);
    for (long long i = threadIdx.x; i < words; i += blockDim.x)
      reinterpret_cast<uint4*>(jsm + s.smem_off)[i] = __ldg(src + i);
  }
  __syncthreads();
  // every loop over steps / stages is fully unrolled with compile-time indices, so the per-stage
  // accumulators and group ids live in registers
  unsigned long long acc[ESC_MAX_STEPS + 1];
#pragma unroll
  for (int i = 0; i <= ESC_MAX_STEPS; ++i) acc[i] = 0;
  const int lane = threadIdx.x & 31;
  const int64_t nwords = (p.nrows + 31) / 32;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < nwords; w += nw) {
    const int64_t row = w * 32 + lane;
    bool sel = row < p.nrows;
    if (sel && p.bitmap != nullptr) sel = (__ldg(p.bitmap + w) >> lane) & 1u;
    if (!sel) continue;
    acc[0] += 1;
    if (p.star) {
      // star: step t is stage t + 1 and its factor is stage-invariant
      unsigned long long run = 1;
#pragma unroll
      for (int t = 0; t < ESC_MAX_STEPS; ++t) {
        if (t >= p.n_steps) break;
        const JoinStepK& s = p.steps[t];
        unsigned long long f = 0;
        if (run != 0 && (s.nulls == nullptr || s.nulls[row] == 0)) {
          const long long k = ld_key(s.keys, s.dtype, row);
          if (s.mode == ESC_JOIN_DENSE) {
            const long long i = k - s.dmin;
            if (i >= 0 && i < s.dlen) f = factor_at(s.smem_off != kNoSmem ? jsm + s.smem_off : s.factor, s.fbits, i);
          } else if (s.mode == ESC_JOIN_PAIRS) {
            f = pairs_find(reinterpret_cast<const longlong2*>(s.slots), s.mask, k,
                           s.smem_off != kNoSmem ? reinterpret_cast<const uint32_t*>(jsm + s.smem_off) : nullptr);
          } else {
            const long long g = hash_find(s.slots, s.mask, s.uk, k);
            if (g >= 0) f = __ldg(s.weight[t + 1] + g);
          }
        }
        run *= f;
        acc[t + 1] += run;
      }
    } else {
      long long g[ESC_MAX_STEPS];
#pragma unroll
      for (int t = 0; t < ESC_MAX_STEPS; ++t) {
        g[t] = -1;
        if (t < p.n_steps) {
          const JoinStepK& s = p.steps[t];
          if (s.nulls == nullptr || s.nulls[row] == 0) g[t] = hash_find(s.slots, s.mask, s.uk, ld_key(s.keys, s.dtype, row));
        }
      }
#pragma unroll
      for (int st = 1; st <= ESC_MAX_STEPS; ++st) {
        if (st > p.n_stages) break;
        unsigned long long prod = 1;
#pragma unroll
        for (int t = 0; t < ESC_MAX_STEPS; ++t) {
          if (t < p.n_steps && p.stage_of[t] <= st)
            prod = g[t] < 0 ? 0ull : prod * (prod ? __ldg(p.steps[t].weight[st] + g[t]) : 0ull);
        }
        acc[st] += prod;
      }
    }
  }
  // block reduction -> one atomicAdd per stage per block
  __shared__ unsigned long long red[kJoinThreads / 32][ESC_MAX_STEPS + 1];
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int st = 0; st <= ESC_MAX_STEPS; ++st) {
    unsigned long long v = acc[st];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) red[warp][st] = v;
  }
  __syncthreads();
  if (threadIdx.x <= p.n_stages) {
    unsigned long long v = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += red[w2][threadIdx.x];
    if (v) atomicAdd(p.out + threadIdx.x, v);
  }
}

// Star over sparse key ranges or wide keys (pair-table, hash or dense steps in any mix): one row
// per thread.  Every step's key is loaded up front (coalesced, all in flight together), so only
// the lookups form the dependent chain; a step is looked up only while the row is alive (issuing
// every step's pair-table lookup at once measured slower: 1.58 vs 1.15 ms, three times the L2
// lookups).  Pair-table lookups test the on-chip occupancy bits first.
template <int NS>
__global__ void __launch_bounds__(kJoinThreads, 2) join_star_kernel(const __grid_constant__ JoinParams p) {
  extern __shared__ __align__(16) uint8_t jsm[];
  for (int t = 0; t < NS; ++t) {
    const JoinStepK& s = p.steps[t];
    if (s.smem_off == kNoSmem) continue;
    const bool pairs = s.mode == ESC_JOIN_PAIRS;
    const long long bytes = pairs ? (long long)((s.mask + 1) / 8)
                                  : s.fbits == 1 ? ((s.dlen + 31) / 32) * 4 : s.dlen * (s.fbits / 8);
    const long long words = (bytes + 15) / 16;
    const uint4* src = reinterpret_cast<const uint4*>(pairs ? reinterpret_cast<const uint8_t*>(s.occ) : s.factor);
    for (long long i = threadIdx.x; i < words; i += blockDim.x)
      reinterpret_cast<uint4*>(jsm + s.smem_off)[i] = __ldg(src + i);
  }
  __syncthreads();
  unsigned long long acc[NS + 1];
#pragma unroll
  for (int i = 0; i <= NS; ++i) acc[i] = 0;
  const int lane = threadIdx.x & 31;
  const int64_t nwords = (p.nrows + 31) / 32;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < nwords; w += nw) {
    const int64_t row = w * 32 + lane;
    bool sel = row < p.nrows;
    if (sel && p.bitmap != nullptr) sel = (__ldg(p.bitmap + w) >> lane) & 1u;
    if (!sel) continue;
    acc[0] += 1;
    long long k[NS];
    bool ok[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const JoinStepK& s = p.steps[t];
      ok[t] = s.nulls == nullptr || s.nulls[row] == 0;
      k[t] = ld_key(s.keys, s.dtype, row);
    }
    unsigned long long run = 1;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const JoinStepK& s = p.steps[t];
      unsigned long long f = 0;
      if (run != 0 && ok[t]) {
        if (s.mode == ESC_JOIN_DENSE) {
          const long long i = k[t] - s.dmin;
          if (i >= 0 && i < s.dlen) f = factor_at(s.smem_off != kNoSmem ? jsm + s.smem_off : s.factor, s.fbits, i);
        } else if (s.mode == ESC_JOIN_PAIRS) {
          f = pairs_find(reinterpret_cast<const longlong2*>(s.slots), s.mask, k[t],
                         s.smem_off != kNoSmem ? reinterpret_cast<const uint32_t*>(jsm + s.smem_off) : nullptr);
        } else {
          const long long g = hash_find(s.slots, s.mask, s.uk, k[t]);
          f = g >= 0 ? __ldg(s.weight[t + 1] + g) : 0ull;
        }
      }
      run *= f;
      acc[t + 1] += run;
    }
  }
  __shared__ unsigned long long red[kJoinThreads / 32][NS + 1];
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int st = 0; st <= NS; ++st) {
    unsigned long long v = acc[st];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) red[warp][st] = v;
  }
  __syncthreads();
  if (threadIdx.x <= NS) {
    unsigned long long v = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += red[w2][threadIdx.x];
    if (v) atomicAdd(p.out + threadIdx.x, v);
  }
}

// Semi-join star (every step a 1-bit dense factor over int32 keys without NULLs — the primary-key
// dimensions of a star schema): a thread owns 4 consecutive rows, issues every step's 16-byte key
// load at once, and walks a 4-bit survivor mask through the on-chip bitmaps; stage s adds
// popc(mask).  No multiplies, 32-bit counters, no dependent global loads.
template <int NS>
__device__ __forceinline__ void bits_load(const JoinParams& p, int64_t q, int64_t full, uint32_t m, int4 (&k)[NS]) {
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    const int* kp = reinterpret_cast<const int*>(p.steps[t].keys);
    if (q < full) {
      k[t] = __ldg(reinterpret_cast<const int4*>(kp) + q);
    } else {  // ragged tail: only the rows that exist
      const int64_t row0 = q * 4;
      k[t].x = (m & 1u) ? __ldg(kp + row0) : 0;
      k[t].y = (m >> 1) & 1u ? __ldg(kp + row0 + 1) : 0;
      k[t].z = (m >> 2) & 1u ? __ldg(kp + row0 + 2) : 0;
      k[t].w = (m >> 3) & 1u ? __ldg(kp + row0 + 3) : 0;
    }
  }
}

template <int NS>
__device__ __forceinline__ uint32_t bits_rows_mask(const JoinParams& p, int64_t q, int64_t full) {
  if (q * 4 >= p.nrows) return 0;
  const int64_t row0 = q * 4;
  uint32_t m = q < full ? 0xFu : (0xFu >> (4 - (p.nrows - row0)));
  if (p.bitmap != nullptr) m &= (__ldg(p.bitmap + (row0 >> 5)) >> (row0 & 31)) & 0xFu;
  return m;
}

template <int NS>
__global__ void __launch_bounds__(kJoinThreads, NS <= 4 ? 2 : 1) join_bits_kernel(const __grid_constant__ JoinParams p) {
  extern __shared__ __align__(16) uint8_t jsm[];
  for (int t = 0; t < NS; ++t) {
    const JoinStepK& s = p.steps[t];
    if (s.smem_off == kNoSmem) continue;
    const long long words = (((s.dlen + 31) / 32) * 4 + 15) / 16;
    for (long long i = threadIdx.x; i < words; i += blockDim.x)
      reinterpret_cast<uint4*>(jsm + s.smem_off)[i] = __ldg(reinterpret_cast<const uint4*>(s.factor) + i);
    if (threadIdx.x == 0) reinterpret_cast<uint4*>(jsm + s.smem_off)[words] = make_uint4(0u, 0u, 0u, 0u);
  }
  __syncthreads();
  uint32_t acc[ESC_MAX_STEPS + 1];
#pragma unroll
  for (int i = 0; i <= ESC_MAX_STEPS; ++i) acc[i] = 0;
  // per-step lookup state in registers: shared-memory bitmap, 32-bit key offset and span
  const uint32_t* bmap[NS];
  int kmin[NS];
  uint32_t klen[NS];
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    bmap[t] = reinterpret_cast<const uint32_t*>(jsm + p.steps[t].smem_off);
    kmin[t] = (int)p.steps[t].dmin;
    klen[t] = (uint32_t)p.steps[t].dlen;
  }
  const int64_t nquads = (p.nrows + 3) / 4;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t full = p.nrows / 4;
  // software pipeline: the next quad's keys are in flight while this quad's masks are computed
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t m = bits_rows_mask<NS>(p, q, full);
  int4 k[NS];
  if (m) bits_load<NS>(p, q, full, m, k);
  while (q < nquads) {
    const int64_t qn = q + nth;
    const uint32_t mn = bits_rows_mask<NS>(p, qn, full);
    int4 kn[NS];
    if (mn) bits_load<NS>(p, qn, full, mn, kn);
    if (m) {
      acc[0] += __popc(m);
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        const int kv[4] = {k[t].x, k[t].y, k[t].z, k[t].w};
        uint32_t hit = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // out of span (a key below min wraps) -> bit klen, a zero bit of the padding; rows
          // outside m are masked below, so no per-row predicate
          const uint32_t i = min((uint32_t)kv[j] - (uint32_t)kmin[t], klen[t]);
          hit |= ((bmap[t][i >> 5] >> (i & 31)) & 1u) << j;
        }
        m &= hit;
        acc[t + 1] += __popc(m);
        if (t + 1 < NS && !__any_sync(__activemask(), m)) break;  // no survivor left among the active lanes
      }
    }
    q = qn;
    m = mn;
#pragma unroll
    for (int t = 0; t < NS; ++t) k[t] = kn[t];
  }
  __shared__ unsigned long long red[kJoinThreads / 32][ESC_MAX_STEPS + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int st = 0; st <= ESC_MAX_STEPS; ++st) {
    unsigned long long v = acc[st];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) red[warp][st] = v;
  }
  __syncthreads();
  if (threadIdx.x <= p.n_stages) {
    unsigned long long v = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += red[w2][threadIdx.x];
    if (v) atomicAdd(p.out + threadIdx.x, v);
  }
}

// Dense-factor star (any integer key widths, NULL keys, factors of any width): a thread owns 4
// consecutive rows; every step's 4 keys are loaded up front (16/32-byte vector loads for
// int32/int64 keys) and the per-row stage products stay in registers.  (Its hash branch is kept
// for completeness; stars with hash steps run join_count_kernel, which measured faster.)
__device__ __forceinline__ void quad_keys(const JoinStepK& s, int64_t row0, int64_t nrows, bool full,
                                          long long (&k)[4], uint32_t& valid) {
  if (full && s.dtype == ESC_I32) {
    const int4 v = __ldg(reinterpret_cast<const int4*>(s.keys) + (row0 >> 2));
    k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
  } else if (full && s.dtype == ESC_I64) {
    const longlong2 a = __ldg(reinterpret_cast<const longlong2*>(s.keys) + (row0 >> 1));
    const longlong2 b = __ldg(reinterpret_cast<const longlong2*>(s.keys) + (row0 >> 1) + 1);
    k[0] = a.x; k[1] = a.y; k[2] = b.x; k[3] = b.y;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) k[j] = row0 + j < nrows ? ld_key(s.keys, s.dtype, row0 + j) : 0;
  }
  if (s.nulls != nullptr) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (row0 + j < nrows && s.nulls[row0 + j]) valid &= ~(1u << j);
  }
}

// Star COUNT probe with small dense factors (every step 1-bit or 8-bit, int32 keys without NULLs,
// factors in shared memory): join_bits_kernel's quad/pipelined structure with a running product
// per row instead of a survivor mask, so dimensions with duplicate keys (8-bit group sizes) stay
// on the fast path; the warp leaves the step chain once every product is zero.
template <int NS>
__global__ void __launch_bounds__(kJoinThreads, NS <= 4 ? 2 : 1) join_small_kernel(const __grid_constant__ JoinParams p) {
  extern __shared__ __align__(16) uint8_t jsm[];
  for (int t = 0; t < NS; ++t) {
    const JoinStepK& s = p.steps[t];
    const long long bytes = s.fbits == 1 ? ((s.dlen + 31) / 32) * 4 : s.dlen;
    const long long words = (bytes + 15) / 16;
    for (long long i = threadIdx.x; i < words; i += blockDim.x)
      reinterpret_cast<uint4*>(jsm + s.smem_off)[i] = __ldg(reinterpret_cast<const uint4*>(s.factor) + i);
    if (threadIdx.x == 0) reinterpret_cast<uint4*>(jsm + s.smem_off)[words] = make_uint4(0u, 0u, 0u, 0u);
  }
  __syncthreads();
  unsigned long long acc[ESC_MAX_STEPS + 1];
#pragma unroll
  for (int i = 0; i <= ESC_MAX_STEPS; ++i) acc[i] = 0;
  const uint8_t* fac[NS];
  int kmin[NS];
  uint32_t klen[NS];
  bool one_bit[NS];
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    fac[t] = jsm + p.steps[t].smem_off;
    kmin[t] = (int)p.steps[t].dmin;
    klen[t] = (uint32_t)p.steps[t].dlen;
    one_bit[t] = p.steps[t].fbits == 1;
  }
  const int64_t nquads = (p.nrows + 3) / 4;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t full = p.nrows / 4;
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t m = bits_rows_mask<NS>(p, q, full);
  int4 k[NS];
  if (m) bits_load<NS>(p, q, full, m, k);
  while (q < nquads) {
    const int64_t qn = q + nth;
    const uint32_t mn = bits_rows_mask<NS>(p, qn, full);
    int4 kn[NS];
    if (mn) bits_load<NS>(p, qn, full, mn, kn);
    if (m) {
      acc[0] += __popc(m);
      unsigned long long run[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) run[j] = (m >> j) & 1u;
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        const int kv[4] = {k[t].x, k[t].y, k[t].z, k[t].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // out of span (a key below min wraps) -> entry klen, a zero of the padding line; a dead
          // row's product stays 0, so no per-row predicate
          const uint32_t i = min((uint32_t)kv[j] - (uint32_t)kmin[t], klen[t]);
          const uint32_t f = one_bit[t] ? (reinterpret_cast<const uint32_t*>(fac[t])[i >> 5] >> (i & 31)) & 1u : fac[t][i];
          run[j] *= f;
        }
        acc[t + 1] += run[0] + run[1] + run[2] + run[3];
        if (t + 1 < NS && !__any_sync(__activemask(), (run[0] | run[1] | run[2] | run[3]) != 0)) break;
      }
    }
    q = qn;
    m = mn;
#pragma unroll
    for (int t = 0; t < NS; ++t) k[t] = kn[t];
  }
  __shared__ unsigned long long red[kJoinThreads / 32][ESC_MAX_STEPS + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int st = 0; st <= ESC_MAX_STEPS; ++st) {
    unsigned long long v = acc[st];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) red[warp][st] = v;
  }
  __syncthreads();
  if (threadIdx.x <= p.n_stages) {
    unsigned long long v = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += red[w2][threadIdx.x];
    if (v) atomicAdd(p.out + threadIdx.x, v);
  }
}

template <int NS>
__global__ void __launch_bounds__(kJoinThreads, 1) join_quad_kernel(const __grid_constant__ JoinParams p) {
  extern __shared__ __align__(16) uint8_t jsm[];
  for (int t = 0; t < NS; ++t) {
    const JoinStepK& s = p.steps[t];
    if (s.mode != ESC_JOIN_DENSE || s.smem_off == kNoSmem) continue;
    const long long bytes = s.fbits == 1 ? ((s.dlen + 31) / 32) * 4 : s.dlen * (s.fbits / 8);
    const long long words = (bytes + 15) / 16;
    for (long long i = threadIdx.x; i < words; i += blockDim.x)
      reinterpret_cast<uint4*>(jsm + s.smem_off)[i] = __ldg(reinterpret_cast<const uint4*>(s.factor) + i);
  }
  __syncthreads();
  unsigned long long acc[NS + 1];
#pragma unroll
  for (int i = 0; i <= NS; ++i) acc[i] = 0;
  const int64_t nquads = (p.nrows + 3) / 4;
  const int64_t full_q = p.nrows / 4;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nquads; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row0 = q * 4;
    const bool full = q < full_q;
    uint32_t sel = full ? 0xFu : (0xFu >> (4 - (p.nrows - row0)));
    if (p.bitmap != nullptr) sel &= (__ldg(p.bitmap + (row0 >> 5)) >> (row0 & 31)) & 0xFu;
    if (sel == 0) continue;
    long long k[NS][4];
    uint32_t valid[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      valid[t] = sel;
      quad_keys(p.steps[t], row0, p.nrows, full, k[t], valid[t]);
    }
    acc[0] += __popc(sel);
    unsigned long long run[4] = {1, 1, 1, 1};
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const JoinStepK& s = p.steps[t];
      unsigned long long f[4] = {0, 0, 0, 0};
      if (s.mode == ESC_JOIN_DENSE) {
        const uint8_t* base = s.smem_off != kNoSmem ? jsm + s.smem_off : s.factor;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const long long i = k[t][j] - s.dmin;
          if (((valid[t] >> j) & 1u) && run[j] != 0 && i >= 0 && i < s.dlen) f[j] = factor_at(base, s.fbits, i);
        }
      } else {
        // interleaved probes: the 4 rows' slot loads are independent
        unsigned long long pos[4];
        long long slot[4];
        bool open[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          open[j] = ((valid[t] >> j) & 1u) && run[j] != 0;
          pos[j] = splitmix64((unsigned long long)k[t][j]) & s.mask;
        }
        bool any = open[0] || open[1] || open[2] || open[3];
        while (any) {
#pragma unroll
          for (int j = 0; j < 4; ++j) slot[j] = open[j] ? __ldg(s.slots + pos[j]) : -1;
          any = false;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (!open[j]) continue;
            if (slot[j] < 0) { open[j] = false; continue; }
            if (__ldg(s.uk + slot[j]) == k[t][j]) {
              f[j] = __ldg(s.weight[t + 1] + slot[j]);
              open[j] = false;
              continue;
            }
            pos[j] = (pos[j] + 1) & s.mask;
            any = true;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) run[j] *= f[j];
      acc[t + 1] += run[0] + run[1] + run[2] + run[3];
    }
  }
  __shared__ unsigned long long red[kJoinThreads / 32][ESC_MAX_STEPS + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int st = 0; st <= NS; ++st) {
    unsigned long long v = acc[st];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) red[warp][st] = v;
  }
  __syncthreads();
  if (threadIdx.x <= NS) {
    unsigned long long v = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += red[w2][threadIdx.x];
    if (v) atomicAdd(p.out + threadIdx.x, v);
  }
}

// ---- hash build grouping (esc_hash_build) ----------------------------------------------------
// 64-bit keys sort as unsigned values with the sign bit flipped (order-preserving)
__global__ void build_gather_kernel(const uint8_t* __restrict__ keys, int dtype, int width,
                                    const int64_t* __restrict__ rows, int64_t n,
                                    unsigned long long* __restrict__ out_keys, int64_t* __restrict__ out_rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows ? rows[i] : i;
    out_keys[i] = (unsigned long long)ld_int(keys + (size_t)r * width, dtype) ^ (1ull << 63);
    out_rows[i] = r;
  }
}

// keys of <= 4 bytes sort as 32-bit unsigned values biased by 2^31 (signed types): the radix sort
// then runs 4 digit passes instead of 8
__global__ void build_gather32_kernel(const uint8_t* __restrict__ keys, int dtype, int width,
                                      const int64_t* __restrict__ rows, int64_t n, uint32_t bias,
                                      uint32_t* __restrict__ out_keys, int64_t* __restrict__ out_rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows ? rows[i] : i;
    out_keys[i] = (uint32_t)ld_int(keys + (size_t)r * width, dtype) + bias;
    out_rows[i] = r;
  }
}

// The whole grouping of a small build (<= 1024 * ITEMS rows, keys of <= 4 bytes) in ONE block:
// a stable block radix sort of the biased 32-bit keys with their rows, group starts by comparing
// neighbours, a block scan for the group ids, then offsets, sizes, unique keys and statistics —
// one launch where the device-wide path costs about a dozen.
constexpr int kBuildSmallThreads = 1024;
template <int ITEMS>
struct BuildSmall {
  using Sort = cub::BlockRadixSort<uint32_t, kBuildSmallThreads, ITEMS, int64_t>;
  using Scan = cub::BlockScan<int, kBuildSmallThreads>;
  using Reduce = cub::BlockReduce<long long, kBuildSmallThreads>;
  using ReduceU = cub::BlockReduce<uint32_t, kBuildSmallThreads>;
  union Temp {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
    typename Reduce::TempStorage reduce;
    typename ReduceU::TempStorage reduce_u;
  };
  static constexpr size_t kSmem = sizeof(Temp) + sizeof(uint32_t) * kBuildSmallThreads;
};

template <int ITEMS>
__global__ void __launch_bounds__(kBuildSmallThreads, 1)
build_small_kernel(const uint8_t* __restrict__ keys, int dtype, int width, const int64_t* __restrict__ rows,
                   int64_t n, uint32_t bias, int64_t* __restrict__ group_rows, long long* __restrict__ uk,
                   long long* __restrict__ counts, long long* __restrict__ start, int64_t* __restrict__ stats) {
  using B = BuildSmall<ITEMS>;
  extern __shared__ __align__(16) uint8_t bsm[];
  typename B::Temp& tmp = *reinterpret_cast<typename B::Temp*>(bsm);
  uint32_t* last_key = reinterpret_cast<uint32_t*>(bsm + sizeof(typename B::Temp));  // per thread
  const int t = threadIdx.x;
  uint32_t k[ITEMS];
  int64_t v[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = (int64_t)t * ITEMS + i;
    if (idx < n) {
      const int64_t r = rows ? rows[idx] : idx;
      k[i] = (uint32_t)ld_int(keys + (size_t)r * width, dtype) + bias;
      v[i] = r;
    } else {
      k[i] = 0xFFFFFFFFu;  // padding: stable, so it stays behind every real row with the same key
      v[i] = -1;
    }
  }
  // sort only the bits the keys span: offsets from the block's smallest key, padding at the top
  // of the range (stable: it stays behind every real row with the same offset).  A dimension's
  // keys span a few thousand values, so the block sort makes 3 passes of 4 bits instead of 8
  __shared__ uint32_t s_lo, s_hi;
  {
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if ((int64_t)t * ITEMS + i < n) {
        lo = min(lo, k[i]);
        hi = max(hi, k[i]);
      }
    const uint32_t blo = typename B::ReduceU(tmp.reduce_u).Reduce(lo, cub::Min());
    __syncthreads();
    const uint32_t bhi = typename B::ReduceU(tmp.reduce_u).Reduce(hi, cub::Max());
    if (t == 0) {
      s_lo = blo;
      s_hi = bhi;
    }
    __syncthreads();
  }
  const uint32_t klo = s_lo;
  const uint32_t span = s_hi - klo;
  const int end_bit = span == 0 ? 1 : 32 - __clz(span);
  const uint32_t pad = end_bit >= 32 ? 0xFFFFFFFFu : ((1u << end_bit) - 1u);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) k[i] = (int64_t)t * ITEMS + i < n ? k[i] - klo : pad;
  typename B::Sort(tmp.sort).Sort(k, v, 0, end_bit);  // blocked arrangement, ascending, stable
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) k[i] += klo;  // (padding wraps harmlessly: never read as a key)
  last_key[t] = k[ITEMS - 1];
  __syncthreads();
  int flag[ITEMS];
  int nf = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t p = (int64_t)t * ITEMS + i;
    const uint32_t prev = i > 0 ? k[i - 1] : (t > 0 ? last_key[t - 1] : 0u);
    flag[i] = (p < n && (p == 0 || k[i] != prev)) ? 1 : 0;
    nf += flag[i];
  }
  int g0, total;
  typename B::Scan(tmp.scan).ExclusiveSum(nf, g0, total);
  int g = g0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t p = (int64_t)t * ITEMS + i;
    if (p < n) group_rows[p] = v[i];
    if (flag[i]) {
      uk[g] = bias ? (long long)(int32_t)(k[i] - bias) : (long long)k[i];
      start[g] = p;
      ++g;
    }
  }
  if (t == 0) start[total] = n;
  __syncthreads();  // every group start is written (global, same block)
  long long most = 0;
  for (int gg = t; gg < total; gg += kBuildSmallThreads) {
    const long long c = __ldcg(start + gg + 1) - __ldcg(start + gg);
    counts[gg] = c;
    most = c > most ? c : most;
  }
  __syncthreads();
  most = typename B::Reduce(tmp.reduce).Reduce(most, cub::Max());
  if (t == 0) {
    stats[0] = total;
    stats[1] = total > 0 ? __ldcg(uk) : 0;
    stats[2] = total > 0 ? __ldcg(uk + total - 1) : 0;
    stats[3] = most;
  }
}

// dense factor array of a star step: bit / count of every key's group at key - lo
__global__ void factor_array_kernel(const long long* __restrict__ unique_keys, const long long* __restrict__ counts,
                                    int64_t u, long long lo, int bits, uint8_t* __restrict__ out) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < u; g += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long i = (unsigned long long)(unique_keys[g] - lo);
    const long long c = counts[g];
    switch (bits) {
      case 1: atomicOr(reinterpret_cast<unsigned int*>(out) + (i >> 5), 1u << (i & 31)); break;
      case 8: out[i] = (uint8_t)c; break;
      case 16: reinterpret_cast<uint16_t*>(out)[i] = (uint16_t)c; break;
      case 32: reinterpret_cast<uint32_t*>(out)[i] = (uint32_t)c; break;
      default: reinterpret_cast<unsigned long long*>(out)[i] = (unsigned long long)c; break;
    }
  }
}

// (key, factor) pair tables of star steps over sparse key ranges
__global__ void pairs_insert_kernel(const long long* __restrict__ uk, const long long* __restrict__ counts, int64_t u,
                                    unsigned long long* pairs, unsigned long long mask, uint32_t* occ) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < u; g += (int64_t)gridDim.x * blockDim.x) {
    const long long key = uk[g];
    const unsigned long long f = (unsigned long long)counts[g];  // >= 1
    unsigned long long h = splitmix64((unsigned long long)key) & mask;
    while (atomicCAS(pairs + 2 * h + 1, 0ull, f) != 0ull) h = (h + 1) & mask;
    pairs[2 * h] = (unsigned long long)key;
    atomicOr(occ + (h >> 5), 1u << (h & 31));
  }
}

struct BuildTemp {  // esc_hash_build's scratch: gathered keys / rows, sorted keys, the sort's own temp
  size_t keys_in, rows_in, keys_sorted, sort, total;
  size_t sort_bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline int build_temp_layout(int64_t n, BuildTemp* T) {
  T->sort_bytes = esc_sort_temp_bytes(n, 8, 1);  // the 64-bit layout also covers 32-bit keys
  size_t off = 0;
  T->keys_in = off;     off += align256((size_t)n * 8);
  T->rows_in = off;     off += align256((size_t)n * 8);
  T->keys_sorted = off; off += align256((size_t)n * 8);
  T->sort = off;        off += align256(T->sort_bytes);
  T->total = off;
  return ESC_OK;
}

}  // namespace esc

// ==========================================================================================
// C ABI (joins)
// ==========================================================================================
extern "C" {

int esc_factor_array(const int64_t* unique_keys, const int64_t* counts, int64_t u, int64_t lo, int64_t span,
                     int32_t bits, void* out, size_t out_bytes, void* stream) {
  if (u < 0 || span < 0 || (bits != 1 && bits != 8 && bits != 16 && bits != 32 && bits != 64))
    return fail(ESC_ERR_INVALID, "bad factor array arguments");
  if ((size_t)((span * bits + 7) / 8) > out_bytes) return fail(ESC_ERR_INVALID, "factor array buffer too small");
  if (out == nullptr || (u > 0 && (unique_keys == nullptr || counts == nullptr)))
    return fail(ESC_ERR_INVALID, "null factor array buffers");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(out, 0, out_bytes, st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("factor array init: ") + cudaGetErrorString(e));
  if (u == 0) return ESC_OK;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (u + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  ++g_launches;
  esc::factor_array_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const long long*>(unique_keys),
                                                             reinterpret_cast<const long long*>(counts), u, lo, bits,
                                                             static_cast<uint8_t*>(out));
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("factor array launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

size_t esc_pairs_bytes(int64_t capacity) {
  if (capacity <= 0) return 0;
  const size_t occ = ((size_t)capacity / 8 + 15) & ~(size_t)15;
  return (size_t)capacity * 16 + (occ < 16 ? 16 : occ);
}

int esc_pairs_build(const int64_t* unique_keys, const int64_t* counts, int64_t u, int64_t* pairs, int64_t capacity,
                    void* stream) {
  if (capacity <= 0 || (capacity & (capacity - 1)) != 0) return fail(ESC_ERR_INVALID, "capacity must be a power of two");
  if (u < 0 || u >= capacity) return fail(ESC_ERR_INVALID, "capacity must exceed the unique keys");
  if (pairs == nullptr || (u > 0 && (unique_keys == nullptr || counts == nullptr)))
    return fail(ESC_ERR_INVALID, "null pair table buffers");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the pairs, then the occupancy bits (capacity / 8 bytes, at least one 16-byte line)
  cudaError_t e = cudaMemsetAsync(pairs, 0, esc_pairs_bytes(capacity), st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("pair table init: ") + cudaGetErrorString(e));
  if (u == 0) return ESC_OK;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (u + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  ++g_launches;
  esc::pairs_insert_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const long long*>(unique_keys),
                                                             reinterpret_cast<const long long*>(counts), u,
                                                             reinterpret_cast<unsigned long long*>(pairs),
                                                             (unsigned long long)capacity - 1,
                                                             reinterpret_cast<uint32_t*>(pairs + 2 * capacity));
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("pair table launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_hash_build_temp_bytes(int64_t n, size_t* bytes) {
  if (bytes == nullptr || n < 0 || n >= (1ll << 31)) return fail(ESC_ERR_INVALID, "bad hash build size");
  esc::BuildTemp T;
  const int rc = esc::build_temp_layout(n, &T);
  if (rc == ESC_OK) *bytes = T.total;
  return rc;
}

int esc_hash_build(const void* keys, int32_t key_dtype, const int64_t* rows, int64_t n, int64_t* out_group_rows,
                   int64_t* out_unique_keys, int64_t* out_group_counts, int64_t* out_group_start, int64_t* out_stats,
                   void* d_temp, size_t temp_bytes, void* stream) {
  if (n < 0 || n >= (1ll << 31)) return fail(ESC_ERR_INVALID, "bad hash build size");
  if (key_dtype == ESC_F32 || key_dtype == ESC_F64 || dtype_width(key_dtype) == 0)
    return fail(ESC_ERR_UNSUPPORTED, "hash keys must be integer columns");
  if (out_stats == nullptr || out_group_start == nullptr || out_group_counts == nullptr ||
      (n > 0 && (keys == nullptr || out_group_rows == nullptr || out_unique_keys == nullptr || d_temp == nullptr)))
    return fail(ESC_ERR_INVALID, "null hash build buffers");
  esc::BuildTemp T;
  int rc = esc::build_temp_layout(n, &T);
  if (rc != ESC_OK) return rc;
  if (n > 0 && temp_bytes < T.total) return fail(ESC_ERR_WORKSPACE, "hash build temp too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* t = static_cast<uint8_t*>(d_temp);
  // one block up to 8K rows: a 16K-row one-block sort (16 items per thread) took 148 us on config
  // 3's part build, the device-wide sort ~40 (query 1.04 -> 0.94 ms; tools/diag_query3.py)
  const bool small_path = dtype_width(key_dtype) <= 4 && n > 0 && n <= (int64_t)esc::kBuildSmallThreads * 8;
  cudaError_t e = cudaSuccess;
  if (n == 0) e = cudaMemsetAsync(out_stats, 0, 4 * sizeof(int64_t), st);
  if (e == cudaSuccess && n == 0) e = cudaMemsetAsync(out_group_start, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("hash build init: ") + cudaGetErrorString(e));
  if (n == 0) return ESC_OK;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  const int w = dtype_width(key_dtype);
  const bool sgn = key_dtype == ESC_I8 || key_dtype == ESC_I16 || key_dtype == ESC_I32;
  if (small_path) {  // one block does it all
    const uint32_t bias = sgn ? 0x80000000u : 0u;
    static std::atomic<int> configured{0};  // bit per instantiation: the attribute is set once
    auto run = [&](auto kern, size_t smem, int bit) -> cudaError_t {
      if (!(configured.load() & bit)) {
        const cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e2 != cudaSuccess) return e2;
        configured.fetch_or(bit);
      }
      ++g_launches;
      kern<<<1, esc::kBuildSmallThreads, smem, st>>>(static_cast<const uint8_t*>(keys), key_dtype, w, rows, n, bias,
                                                     out_group_rows, reinterpret_cast<long long*>(out_unique_keys),
                                                     reinterpret_cast<long long*>(out_group_counts),
                                                     reinterpret_cast<long long*>(out_group_start), out_stats);
      return cudaGetLastError();
    };
    // the fewest items per thread that hold the build (a smaller block sort per launch)
    e = n <= esc::kBuildSmallThreads     ? run(esc::build_small_kernel<1>, esc::BuildSmall<1>::kSmem, 1)
        : n <= 2 * esc::kBuildSmallThreads ? run(esc::build_small_kernel<2>, esc::BuildSmall<2>::kSmem, 2)
        : n <= 4 * esc::kBuildSmallThreads ? run(esc::build_small_kernel<4>, esc::BuildSmall<4>::kSmem, 4)
                                           : run(esc::build_small_kernel<8>, esc::BuildSmall<8>::kSmem, 8);
    if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("small hash build: ") + cudaGetErrorString(e));
    return ESC_OK;
  }
  // the framework's own stable LSD radix sort (esc_sort.cuh): equal keys keep ascending build-row
  // order, as the reference's stable argsort; then the runs are the groups in ascending key order
  uint8_t* ks = t + T.keys_sorted;
  int64_t* rows_in = reinterpret_cast<int64_t*>(t + T.rows_in);
  if (w <= 4) {  // 32-bit keys (biased by 2^31 when signed): 4 digit passes instead of 8
    const uint32_t bias = sgn ? 0x80000000u : 0u;
    uint32_t* k32_in = reinterpret_cast<uint32_t*>(t + T.keys_in);
    ++g_launches;
    esc::build_gather32_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const uint8_t*>(keys), key_dtype, w,
                                                                 rows, n, bias, k32_in, rows_in);
    rc = esc_sort_pairs(k32_in, reinterpret_cast<const uint64_t*>(rows_in), ks,
                        reinterpret_cast<uint64_t*>(out_group_rows), n, 4, 0, 32, t + T.sort, T.sort_bytes, st);
    if (rc == ESC_OK)
      rc = esc_runs(ks, 4, sgn ? esc::ESC_KEY_I32 : esc::ESC_KEY_RAW, n, out_unique_keys, out_group_start,
                    out_group_counts, nullptr, out_stats, t + T.sort, T.sort_bytes, st);
  } else {
    unsigned long long* k64_in = reinterpret_cast<unsigned long long*>(t + T.keys_in);
    ++g_launches;
    esc::build_gather_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const uint8_t*>(keys), key_dtype, w, rows,
                                                               n, k64_in, rows_in);
    rc = esc_sort_pairs(k64_in, reinterpret_cast<const uint64_t*>(rows_in), ks,
                        reinterpret_cast<uint64_t*>(out_group_rows), n, 8, 0, 64, t + T.sort, T.sort_bytes, st);
    if (rc == ESC_OK)
      rc = esc_runs(ks, 8, esc::ESC_KEY_I64, n, out_unique_keys, out_group_start, out_group_counts, nullptr,
                    out_stats, t + T.sort, T.sort_bytes, st);
  }
  return rc;
}

int esc_hash_insert(const int64_t* unique_keys, int64_t n_unique, int64_t* slots, int64_t capacity, void* stream) {
  if (capacity <= 0 || (capacity & (capacity - 1)) != 0) return fail(ESC_ERR_INVALID, "capacity must be a power of two");
  if (n_unique < 0 || n_unique >= capacity) return fail(ESC_ERR_INVALID, "capacity must exceed the unique keys");
  if (slots == nullptr || (n_unique > 0 && unique_keys == nullptr)) return fail(ESC_ERR_INVALID, "null hash buffers");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(slots, 0xFF, (size_t)capacity * sizeof(int64_t), st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("slot init: ") + cudaGetErrorString(e));
  if (n_unique == 0) return ESC_OK;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (n_unique + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  ++g_launches;
  esc::hash_insert_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const long long*>(unique_keys), n_unique,
                                                            reinterpret_cast<unsigned long long*>(slots),
                                                            (unsigned long long)capacity - 1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("hash insert launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_hash_probe(const int64_t* slots, int64_t capacity, const int64_t* unique_keys, const void* keys,
                   int32_t key_dtype, const uint8_t* key_nulls, const int64_t* rows, const uint8_t* valid, int64_t n,
                   int64_t* out_groups, void* stream) {
  if (capacity <= 0 || (capacity & (capacity - 1)) != 0) return fail(ESC_ERR_INVALID, "capacity must be a power of two");
  if (n < 0) return fail(ESC_ERR_INVALID, "negative probe count");
  if (n == 0) return ESC_OK;
  if (slots == nullptr || unique_keys == nullptr || keys == nullptr || out_groups == nullptr)
    return fail(ESC_ERR_INVALID, "null probe buffers");
  if (key_dtype == ESC_F32 || key_dtype == ESC_F64 || dtype_width(key_dtype) == 0)
    return fail(ESC_ERR_UNSUPPORTED, "hash keys must be integer columns");
  esc::ProbeParams p;
  p.slots = reinterpret_cast<const long long*>(slots);
  p.mask = (unsigned long long)capacity - 1;
  p.uk = reinterpret_cast<const long long*>(unique_keys);
  p.keys = static_cast<const uint8_t*>(keys);
  p.dtype = key_dtype;
  p.nulls = key_nulls;
  p.rows = rows;
  p.valid = valid;
  p.n = n;
  p.out = reinterpret_cast<long long*>(out_groups);
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  ++g_launches;
  esc::hash_probe_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("hash probe launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_expand(const int64_t* groups, const int64_t* offsets, int64_t n, const int64_t* group_start,
               const int64_t* group_rows, int64_t* out_tuple, int64_t* out_row, void* stream) {
  if (n < 0) return fail(ESC_ERR_INVALID, "negative tuple count");
  if (n == 0) return ESC_OK;
  if (groups == nullptr || offsets == nullptr || group_start == nullptr || out_row == nullptr)
    return fail(ESC_ERR_INVALID, "null expansion buffers");
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  ++g_launches;
  esc::expand_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(groups), reinterpret_cast<const long long*>(offsets), n,
      reinterpret_cast<const long long*>(group_start), reinterpret_cast<const long long*>(group_rows),
      reinterpret_cast<long long*>(out_tuple), reinterpret_cast<long long*>(out_row));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("expand launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_join_count(const esc_join_t* j, uint64_t* d_stage_counts, void* stream) {
  if (j == nullptr || d_stage_counts == nullptr) return fail(ESC_ERR_INVALID, "null join arguments");
  if (j->n_steps < 0 || j->n_steps > ESC_MAX_STEPS || j->n_stages < 0 || j->n_stages > ESC_MAX_STEPS)
    return fail(ESC_ERR_INVALID, "join step count out of range");
  if (j->nrows < 0) return fail(ESC_ERR_INVALID, "negative probe rows");
  static thread_local esc::JoinParams p;
  std::memset(&p, 0, sizeof(p));
  p.n_steps = j->n_steps;
  p.n_stages = j->n_stages;
  p.star = j->star ? 1 : 0;
  p.nrows = j->nrows;
  p.bitmap = j->bitmap;
  p.out = reinterpret_cast<unsigned long long*>(d_stage_counts);
  int prev_stage = 0;
  uint32_t smem = 0;
  const uint32_t smem_cap = 160 * 1024;
  for (int t = 0; t < j->n_steps; ++t) {
    const esc_join_step_t& s = j->steps[t];
    esc::JoinStepK& k = p.steps[t];
    if (j->stage_of[t] <= prev_stage || j->stage_of[t] > j->n_stages)
      return fail(ESC_ERR_INVALID, "stage_of must increase within 1..n_stages");
    prev_stage = p.stage_of[t] = j->stage_of[t];
    if (s.key_data == nullptr && j->nrows > 0) return fail(ESC_ERR_INVALID, "null join key column");
    if (s.key_dtype == ESC_F32 || s.key_dtype == ESC_F64 || dtype_width(s.key_dtype) == 0)
      return fail(ESC_ERR_UNSUPPORTED, "join keys must be integer columns");
    k.keys = static_cast<const uint8_t*>(s.key_data);
    k.nulls = s.key_nulls;
    k.dtype = s.key_dtype;
    k.mode = s.mode;
    k.smem_off = esc::kNoSmem;
    if (s.mode == ESC_JOIN_DENSE) {
      if (!j->star) return fail(ESC_ERR_INVALID, "dense factor arrays need a star (stage-invariant) join");
      if (s.factor_bits != 1 && s.factor_bits != 8 && s.factor_bits != 16 && s.factor_bits != 32 && s.factor_bits != 64)
        return fail(ESC_ERR_INVALID, "factor_bits must be 1, 8, 16, 32 or 64");
      if (s.dense_len < 0 || (s.dense_len > 0 && s.factor == nullptr)) return fail(ESC_ERR_INVALID, "bad dense factor");
      if (reinterpret_cast<uintptr_t>(s.factor) % 16 != 0) return fail(ESC_ERR_INVALID, "factor array must be 16-byte aligned");
      k.dmin = s.dense_min;
      k.dlen = s.dense_len;
      k.factor = static_cast<const uint8_t*>(s.factor);
      k.fbits = s.factor_bits;
      const long long bytes = s.factor_bits == 1 ? ((s.dense_len + 31) / 32) * 4 : s.dense_len * (s.factor_bits / 8);
      // (one zero line after the array: join_bits_kernel / join_small_kernel clamp an out-of-span
      // key to entry dense_len, which must read 0)
      const uint32_t need = (uint32_t)((bytes + 15) / 16 * 16) + 16u;
      if (bytes <= (long long)smem_cap && smem + need <= smem_cap) {
        k.smem_off = smem;
        smem += need;
      }
    } else if (s.mode == ESC_JOIN_PAIRS) {
      if (!j->star) return fail(ESC_ERR_INVALID, "pair tables need a star (stage-invariant) join");
      if (s.capacity <= 0 || (s.capacity & (s.capacity - 1)) != 0 || s.slots == nullptr ||
          reinterpret_cast<uintptr_t>(s.slots) % 16 != 0)
        return fail(ESC_ERR_INVALID, "bad pair table");
      k.slots = reinterpret_cast<const long long*>(s.slots);
      k.mask = (unsigned long long)s.capacity - 1;
      k.occ = reinterpret_cast<const uint32_t*>(s.slots + 2 * s.capacity);
      const uint32_t need = (uint32_t)((((unsigned long long)s.capacity / 8) + 15) / 16 * 16);
      static const bool occ_on = [] { const char* e = getenv("ESC_PAIRS_OCC"); return !(e && e[0] == '0'); }();
      if (occ_on && (long long)s.capacity / 8 <= (long long)smem_cap && smem + need <= smem_cap) {  // occupancy bits on chip
        k.smem_off = smem;
        smem += need;
      }
    } else if (s.mode == ESC_JOIN_HASH) {
      if (s.capacity <= 0 || (s.capacity & (s.capacity - 1)) != 0 || s.slots == nullptr || s.unique_keys == nullptr)
        return fail(ESC_ERR_INVALID, "bad hash table");
      k.slots = reinterpret_cast<const long long*>(s.slots);
      k.mask = (unsigned long long)s.capacity - 1;
      k.uk = reinterpret_cast<const long long*>(s.unique_keys);
      for (int st = p.stage_of[t]; st <= j->n_stages; ++st) {
        if (s.weight[st] == nullptr) return fail(ESC_ERR_INVALID, "missing stage weight array");
        k.weight[st] = reinterpret_cast<const unsigned long long*>(s.weight[st]);
      }
    } else {
      return fail(ESC_ERR_INVALID, "bad join step mode");
    }
  }
  if (j->star && j->n_steps != j->n_stages) return fail(ESC_ERR_INVALID, "a star join probes every stage");
  p.bits = p.star;
  for (int t = 0; t < j->n_steps; ++t) {
    const esc::JoinStepK& k = p.steps[t];
    if (k.mode != ESC_JOIN_DENSE || k.fbits != 1 || k.dtype != ESC_I32 || k.nulls != nullptr ||
        reinterpret_cast<uintptr_t>(k.keys) % 16 != 0 || k.smem_off == esc::kNoSmem || k.dmin < INT32_MIN ||
        k.dmin > INT32_MAX || k.dlen > INT32_MAX)
      p.bits = 0;
  }
  p.smem_bytes = smem;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_stage_counts, 0, (size_t)(j->n_stages + 1) * sizeof(uint64_t), st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("stage count init: ") + cudaGetErrorString(e));
  if (j->nrows == 0) return ESC_OK;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  static void (*const bits_kernels[ESC_MAX_STEPS + 1])(const esc::JoinParams) = {
      nullptr, esc::join_bits_kernel<1>, esc::join_bits_kernel<2>, esc::join_bits_kernel<3>,
      esc::join_bits_kernel<4>, esc::join_bits_kernel<5>, esc::join_bits_kernel<6>, esc::join_bits_kernel<7>,
      esc::join_bits_kernel<8>};
  static void (*const quad_kernels[ESC_MAX_STEPS + 1])(const esc::JoinParams) = {
      nullptr, esc::join_quad_kernel<1>, esc::join_quad_kernel<2>, esc::join_quad_kernel<3>,
      esc::join_quad_kernel<4>, esc::join_quad_kernel<5>, esc::join_quad_kernel<6>, esc::join_quad_kernel<7>,
      esc::join_quad_kernel<8>};
  static void (*const star_kernels[ESC_MAX_STEPS + 1])(const esc::JoinParams) = {
      nullptr, esc::join_star_kernel<1>, esc::join_star_kernel<2>, esc::join_star_kernel<3>,
      esc::join_star_kernel<4>, esc::join_star_kernel<5>, esc::join_star_kernel<6>, esc::join_star_kernel<7>,
      esc::join_star_kernel<8>};
  static void (*const small_kernels[ESC_MAX_STEPS + 1])(const esc::JoinParams) = {
      nullptr, esc::join_small_kernel<1>, esc::join_small_kernel<2>, esc::join_small_kernel<3>,
      esc::join_small_kernel<4>, esc::join_small_kernel<5>, esc::join_small_kernel<6>, esc::join_small_kernel<7>,
      esc::join_small_kernel<8>};
  if (p.n_steps == 0) p.bits = 0;
  // semi-join bitmaps -> join_bits_kernel; 1/8-bit factors over int32 keys -> join_small_kernel;
  // any other all-dense star -> join_quad_kernel; a star with pair-table or hash steps ->
  // join_star_kernel (one row per thread, every step's key loaded up front); snowflake
  // (stage-dependent weights) -> join_count_kernel
  bool quad = !p.bits && p.star && p.n_steps > 0;
  for (int t = 0; t < p.n_steps; ++t)
    if (p.steps[t].mode != ESC_JOIN_DENSE) quad = false;
  bool small = quad;
  for (int t = 0; t < p.n_steps && small; ++t) {
    const esc::JoinStepK& k = p.steps[t];
    small = (k.fbits == 1 || k.fbits == 8) && k.dtype == ESC_I32 && k.nulls == nullptr &&
            reinterpret_cast<uintptr_t>(k.keys) % 16 == 0 && k.smem_off != esc::kNoSmem && k.dmin >= INT32_MIN &&
            k.dmin <= INT32_MAX && k.dlen <= INT32_MAX;
  }
  const bool star1 = !p.bits && !quad && p.star && p.n_steps > 0;
  auto kern = p.bits  ? bits_kernels[p.n_steps]
              : small ? small_kernels[p.n_steps]
              : quad  ? quad_kernels[p.n_steps]
              : star1 ? star_kernels[p.n_steps]
                      : esc::join_count_kernel;
  static thread_local uint32_t configured[4 * ESC_MAX_STEPS + 4] = {};
  const int ci = p.bits ? p.n_steps
                 : small ? 2 * (ESC_MAX_STEPS + 1) + p.n_steps
                 : quad  ? ESC_MAX_STEPS + 1 + p.n_steps
                 : star1 ? 3 * (ESC_MAX_STEPS + 1) + p.n_steps
                         : 0;
  if (smem > 48 * 1024 && smem > configured[ci]) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    configured[ci] = smem;
  }
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, esc::kJoinThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t units = (p.bits || quad) ? (j->nrows + 3) / 4 / 32 + 1 : (j->nrows + 31) / 32;  // warps of work
  int64_t blocks = (units + esc::kJoinThreads / 32 - 1) / (esc::kJoinThreads / 32);
  if (blocks > (int64_t)sms * per_sm) blocks = (int64_t)sms * per_sm;
  if (blocks < 1) blocks = 1;
  ++g_launches;
  kern<<<(unsigned)blocks, esc::kJoinThreads, smem, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("join count launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

}  // extern "C"
