// fs_jit_kernels.cuh -- device helpers for the program-specialised (NVRTC) kernels.
//
// A specialised kernel has every instruction of the bytecode program unrolled in straight-line
// code with constant operands; the frame lives in shared memory at constant offsets
// (physical slots after H/SWAP renaming, which the generator resolves at compile time), so the
// compiler keeps it in registers between noise blocks.  Noise blocks call the helper below with
// the site masks already translated to physical slots.
#pragma once
#include "fs_general.cuh"

namespace fs {

// apply the word's pre-drawn faults of sites < hi, XORing into physical slots:
// pslot[j] = physical frame slot of Pauli entry j under the renaming at its NoiseBlock.
__device__ __noinline__ void jit_noise_block(const DevProg& P, uint32_t* F, const uint16_t* __restrict__ pslot,
                                                FaultBuffer<kFaultCap>& fb, int hi) {
  fb.apply_until(P, hi, [&](int c, int l) {
    const int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
    for (int j = off; j < end; j++) F[(uint32_t)__ldg(pslot + j) * 32] ^= 1u << l;
  });
}

// general kernel: regenerate the word's faults with sites < hi in place (overflowed fault list;
// rare) -- one out-of-line copy instead of one inlined generator per NoiseBlock
__device__ __noinline__ void gjit_noise_fallback(const DevProg& P, uint32_t* Fs, const uint16_t* __restrict__ pslot,
                                                 WordFaultGen& gen, int& psite, int& plane, int& pcase, int hi) {
  for (;;) {
    if (psite < 0) {
      int st_, ln_, cs_;
      const int r_ = gen.step(P, st_, ln_, cs_);
      if (r_ == 2) { psite = 0x7FFFFFFF; break; }
      if (r_ == 0) continue;
      psite = st_; plane = ln_; pcase = cs_;
    }
    if (psite >= hi) break;
    for (int j = __ldg(P.case_pauli_off + pcase); j < __ldg(P.case_pauli_off + pcase + 1); j++)
      Fs[__ldg(pslot + j)] ^= 1u << plane;
    psite = -1;
  }
}

// Noise for the specialised frame kernel.  fault_list_kernel generates each 32-shot word's
// faults (WordFaultGen: the engine stream; lane = word) and writes one entry per fault,
// ent[i][W] = pauli_off << 10 | pauli_cnt << 5 | shot_bit, plus per-NoiseBlock counts
// bcount[b][W] and the total ntot[W].  The frame kernel copies a warp's entries into shared
// memory with full-row (coalesced) loads once per word and applies them from there.  A word
// with more than `cap` faults, or a fault with more than 31 Pauli entries, is marked
// ntot = ~0 and regenerates its stream in place (identical results).
__global__ void __launch_bounds__(256) fault_list_kernel(DevProg P, uint64_t seed, uint64_t word0, uint32_t nw,
                                                        uint32_t W, const int* __restrict__ site_block, int nblocks,
                                                        uint32_t* __restrict__ ent, uint32_t* __restrict__ bcount,
                                                        uint32_t* __restrict__ ntot, uint32_t cap) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;  // W = row stride, nw = words
  if (w >= nw) return;
  WordFaultGen gen;
  gen.init(seed, word0 + w);
  uint32_t n = 0, nb = 0;
  int blk = 0;
  int site = 0, lane = 0, cs = 0;
  bool over = false;
  for (;;) {
    const int r = gen.step(P, site, lane, cs);
    if (r == 2) break;
    if (r == 0) continue;
    const int b = __ldg(site_block + site);
    for (; blk < b; blk++) {
      bcount[(size_t)blk * W + w] = nb;
      nb = 0;
    }
    const int off = __ldg(P.case_pauli_off + cs), cnt = __ldg(P.case_pauli_off + cs + 1) - off;
    if (n == cap || cnt > 31 || off >= (1 << 22)) { over = true; break; }
    ent[(size_t)n * W + w] = ((uint32_t)off << 10) | ((uint32_t)cnt << 5) | (uint32_t)lane;
    n++;
    nb++;
  }
  if (over) {
    ntot[w] = 0xFFFFFFFFu;
    return;
  }
  for (; blk < nblocks; blk++) {
    bcount[(size_t)blk * W + w] = nb;
    nb = 0;
  }
  ntot[w] = n;
}

// apply n staged fault entries (stage[t * 32 + lane]) to the frame
__device__ __forceinline__ void jit_apply_faults(uint32_t* F, const uint32_t* stage, const uint16_t* __restrict__ pslot,
                                                 int lane, uint32_t& cur, uint32_t n) {
  for (uint32_t t = 0; t < n; t++) {
    const uint32_t e = stage[(cur + t) * 32 + lane];
    const uint32_t bit = 1u << (e & 31);
    const int off = (int)(e >> 10), cnt = (int)((e >> 5) & 31);
    // issue the slot lookups of up to 8 entries together (independent L1 loads), then the XORs
    uint32_t sl[8];
#pragma unroll
    for (int j = 0; j < 8; j++) sl[j] = j < cnt ? (uint32_t)__ldg(pslot + off + j) : 0u;
#pragma unroll
    for (int j = 0; j < 8; j++)
      if (j < cnt) F[sl[j] * 32] ^= bit;
    for (int j = 8; j < cnt; j++) F[(uint32_t)__ldg(pslot + off + j) * 32] ^= bit;
  }
  cur += n;
}

__device__ __forceinline__ uint4 coin_block(uint64_t seed, uint64_t wabs, int blk) {
  return philox((uint32_t)wabs, (uint32_t)(wabs >> 32), (uint32_t)blk, TAG_COIN << 24, seed);
}

}  // namespace fs

namespace fs {

// Affine frame kernel (fs_affine.cuh).  Fault tables (shared memory when they fit): rows flipped
// by each case (as buffer slots for word 0), site -> (first case, class), class -> (case count, p,
// cumulative case probabilities), the ln table of the gap draws.
template <bool OFF16>
struct AffTabs {
  const uint16_t* crows;
  const uint32_t* crow_off;  // u16 entries when OFF16
  const uint32_t* site_case;
  const uint16_t* site_cls;
  const int* cls_nc;
  const double* cls_prob;
  const double* cls_cum;
  const double* cls_scale;  // nc / p: first guess of the case index
  const double2* lntab;
  int cw;
  uint32_t dump;  // first of 32 scratch words after the row buffer (multiple of 32)
  __device__ __forceinline__ uint32_t off(int c) const {
    return OFF16 ? (uint32_t)reinterpret_cast<const uint16_t*>(crow_off)[c] : crow_off[c];
  }
};

// One fault: case pick by bisect_right over the class's cumulative case probabilities (clamped),
// then its shot bit XORed into the case's rows of word wi.  Row r of word wi lives at
// slot(r, wi) = r * G + (wi ^ sw(r)) = slot(r, 0) ^ wi (fs_affine.cuh aff_sw): the lanes working on
// one word spread over all 32 banks (shared atomics: two lanes may flip the same row).
template <bool OFF16, bool UNIFORM>
__device__ __forceinline__ int aff_case(const AffTabs<OFF16>& T, int site, int cls, double x) {
#ifdef FS_AFF_CLS_CONST  // class case counts and scales as generated constants (no table loads)
  const int nc = fs_aff_cls_nc(cls);
#else
  const int nc = T.cls_nc[cls];
#endif
  int c = 0;
  if (nc > 1) {
    // bisect_right(cum, x) clamped to nc - 1 == the first c < nc - 1 with x < cum[c], else nc - 1:
    // the uniform-case guess x * nc / p corrected by one step each way, exact bisect if still off
    const double* cum = T.cls_cum + cls * T.cw;
#ifdef FS_AFF_CLS_CONST
    const double y = x * fs_aff_cls_scale(cls);
#else
    const double y = x * T.cls_scale[cls];
#endif
    c = min((int)y, nc - 1);
#ifdef FS_AFF_SAFEZONE
    // every cum[i] * nc / p lies within eps(k) of i + 1 (host-checked, eps >= 1 for classes that do
    // not): a y at least eps away from every integer is already exact, without table loads
    const double fr = y - (double)(int)y;
    if (!(fr >= fs_aff_cls_eps(cls) && fr <= 1.0 - fs_aff_cls_eps(cls)))
#endif
    {
      c -= (c > 0 && x < cum[c - 1]) ? 1 : 0;
      c += (c < nc - 1 && !(x < cum[c])) ? 1 : 0;
      // classes whose cumulative probabilities sit within one bin of the uniform grid (the host
      // checks; e.g. DEPOLARIZE1/2) are exact after the one-step correction
      if (!UNIFORM && ((c > 0 && x < cum[c - 1]) || (c < nc - 1 && !(x < cum[c])))) {
        int lo = 0, hi = nc;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (x < cum[mid]) hi = mid; else lo = mid + 1;
        }
        c = lo < nc - 1 ? lo : nc - 1;
      }
    }
  }
  return (int)T.site_case[site] + c;
}

// case cs -> its row list crows[j0 .. j0 + n)
template <bool OFF16>
__device__ __forceinline__ void aff_case_rows(const AffTabs<OFF16>& T, int cs, uint32_t& j0, uint32_t& n) {
  j0 = T.off(cs);
  n = T.off(cs + 1) - j0;
}

// All lanes together (converged): lane l XORs `bit` into the n rows crows[j0 .. j0 + n) of word wi
// (n = 0: no fault).  The trip count is the warp's largest n; slots past a lane's list go to its own
// dump word (B[dump + lane], never read), so the shared atomics issue without divergence.
template <bool OFF16>
__device__ __forceinline__ void aff_rows(const AffTabs<OFF16>& T, uint32_t* B, uint32_t wi, uint32_t j0, uint32_t n,
                                         uint32_t bit) {
#if defined(FS_AFF_DIAG) && FS_AFF_DIAG == 1
  return;  // diagnostic: no row application
#endif
  const uint32_t nmax = __reduce_max_sync(0xFFFFFFFFu, n);
  const uint32_t dl = T.dump + (threadIdx.x & 31);
  // two rows per trip (the odd tail's second XOR goes to the dump word): half the loop overhead
  for (uint32_t t = 0; t < nmax; t += 2) {
    const uint32_t e0 = t < n ? (uint32_t)T.crows[j0 + t] : dl;
    const uint32_t e1 = t + 1 < n ? (uint32_t)T.crows[j0 + t + 1] : dl;
    atomicXor(B + (e0 ^ wi), bit);
    atomicXor(B + (e1 ^ wi), bit);
  }
}

// Load-balanced form of aff_rows: the warp's fault rows (sum of n over lanes, ~3.7 per fault) are
// spread over the lanes 32 at a time instead of every lane looping to the warp's largest n.  Entry
// t of the concatenated lists belongs to the last lane whose exclusive start is <= t (a lane with
// n = 0 never is: the next lane has the same start); the owner is found by a 5-step binary search
// over the lanes' starts (shuffles).  Same XORs as aff_rows, in another order (XOR commutes).
template <bool OFF16>
__device__ __forceinline__ void aff_rows_bal(const AffTabs<OFF16>& T, uint32_t* B, uint32_t wi, uint32_t j0, uint32_t n,
                                             uint32_t bit) {
#if defined(FS_AFF_DIAG) && FS_AFF_DIAG == 1
  return;  // diagnostic: no row application
#endif
  const int lane = threadIdx.x & 31;
  uint32_t e = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, e, o);
    if (lane >= o) e += t;
  }
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, e, 31);
  const uint32_t s = e - n;                  // exclusive start of this lane's rows
  const uint32_t base = j0 - s;              // row-list index of entry t = base(owner) + t
  for (uint32_t t0 = 0; t0 < total; t0 += 32) {
    const uint32_t t = t0 + (uint32_t)lane;
    int l = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1) {
      const uint32_t sv = __shfl_sync(0xFFFFFFFFu, s, l + step);
      if (sv <= t) l += step;
    }
    const uint32_t b = __shfl_sync(0xFFFFFFFFu, base, l);
    const uint32_t bv = __shfl_sync(0xFFFFFFFFu, bit, l);
    if (t < total) atomicXor(B + ((uint32_t)T.crows[b + t] ^ wi), bv);
  }
}

#ifndef FS_AFF_ROWS
#define FS_AFF_ROWS aff_rows  // measured: the balanced form's shuffles cost more MIO than they save
#endif

// Faults of one 32-shot word, warp-cooperatively: lane j evaluates step st + j of the word's
// noise stream (the WordFaultGen process, step by step the same draws and decisions), the cell
// positions of a run are an inclusive warp scan of the per-step advances 1 + floor(ln(U) * lp), and
// the first step past the run's last cell ends it (the following lanes start the next run).
// Generic over runs (certain sites, several probabilities).
template <bool OFF16, bool UNIFORM>
__device__ __forceinline__ void aff_word_faults(const DevProg& P, const AffTabs<OFF16>& T, uint32_t* B, uint32_t wi,
                                                uint64_t seed, uint64_t wabs, int lane) {
  const int nruns = P.num_runs;
  uint32_t st = 0;
  int run = 0, cl = 0;
  long long c = -1;
  while (run < nruns) {
    const uint4 b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), 0u, (TAG_NOISE << 24) | (st + lane), seed);
    const double u2 = u64_to_unit(((uint64_t)b.w << 32) | b.z);
    const double L = ln_unit_t(((uint64_t)b.y << 32) | b.x, T.lntab);
    int first = 0;
    while (first < 32 && run < nruns) {
      const int start = __ldg(P.run_start + run), len = __ldg(P.run_len + run);
      int site = -1, fl = 0, cls = 0;
      double x = 0.0;
      if (len == 0) {  // certain site: the run's steps fire shot bits cl, cl + 1, ..., 31 in order
        const int take = min(32 - first, 32 - cl);
        if (lane >= first && lane < first + take) {
          site = start;
          fl = cl + lane - first;
          cls = T.site_cls[site];
#ifdef FS_AFF_CLS_CONST
          x = u2 * fs_aff_cls_prob(cls);
#else
          x = u2 * T.cls_prob[cls];
#endif
        }
        cl += take;
        first += take;
        if (cl == 32) { run++; cl = 0; }
      } else {
        long long inc = 0;
        if (lane >= first) {
          const double g = floor(__dmul_rn(L, __ldg(P.run_lp + run)));
          inc = g < 4.0e12 ? (long long)g + 1 : (1LL << 42);
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
          if (lane >= o) inc += t;
        }
        const long long pos = c + inc, limit = 32LL * len;
        const uint32_t endm = __ballot_sync(0xFFFFFFFFu, lane >= first && pos >= limit);
        if (lane >= first && pos < limit) {
          const int s = start + (int)(pos >> 5);
          const double xs = __dmul_rn(u2, __ldg(P.run_q + run));
          const int k = T.site_cls[s];
#ifdef FS_AFF_CLS_CONST
          if (xs < fs_aff_cls_prob(k)) {  // thinning: p_site < q
#else
          if (xs < T.cls_prob[k]) {  // thinning: p_site < q
#endif
            site = s;
            fl = (int)(pos & 31);
            cls = k;
            x = xs;
          }
        }
        if (endm) {
          first = __ffs(endm);  // the lane after the ending step
          run++;
          c = -1;
        } else {
          c = __shfl_sync(0xFFFFFFFFu, pos, 31);
          first = 32;
        }
      }
      uint32_t j0 = 0, n = 0;
      if (site >= 0) aff_case_rows(T, aff_case<OFF16, UNIFORM>(T, site, cls, x), j0, n);
      FS_AFF_ROWS<OFF16>(T, B, wi, j0, n, 1u << fl);
    }
    st += 32;
  }
}

// The common case of one geometric run over all noisy sites (every site of the program has the
// same p up to 1e-9, e.g. a uniform circuit-level noise model) with fewer than 2^25 cells: the
// run parameters stay in registers and the scan is 32-bit.
struct AffRun1 {
  int start;
  uint32_t limit;
  double lp, q;
};

template <bool OFF16, bool UNIFORM>
__device__ __forceinline__ void aff_word_faults_1run(const AffTabs<OFF16>& T, uint32_t* B, uint32_t wi, uint64_t seed,
                                                     uint64_t wabs, int lane, const AffRun1& R) {
  uint32_t st = 0;
  int c = -1;
  for (;;) {
    const uint4 b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), 0u, (TAG_NOISE << 24) | (st + lane), seed);
    const double u2 = u64_to_unit(((uint64_t)b.w << 32) | b.z);
    const double g = floor(__dmul_rn(ln_unit_t(((uint64_t)b.y << 32) | b.x, T.lntab), R.lp));
    int inc = g < 33554432.0 ? (int)g + 1 : 33554432;  // 2^25 >= limit: a clamped step ends the run
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += t;
    }
    const int pos = c + inc;
    const bool in = pos < (int)R.limit;
    const uint32_t endm = __ballot_sync(0xFFFFFFFFu, !in);
    uint32_t j0 = 0, n = 0;
    if (in) {
      const int s = R.start + (pos >> 5);
      const double x = __dmul_rn(u2, R.q);
      const int k = T.site_cls[s];
#ifdef FS_AFF_CLS_CONST  // thinning bound from the generated class constants
      if (x < fs_aff_cls_prob(k)) {
#else
      if (x < T.cls_prob[k]) {  // thinning: p_site < q
#endif
        aff_case_rows(T, aff_case<OFF16, UNIFORM>(T, s, k, x), j0, n);
      }
    }
    FS_AFF_ROWS<OFF16>(T, B, wi, j0, n, 1u << (pos & 31));
    if (endm) return;
    c = __shfl_sync(0xFFFFFFFFu, pos, 31);
    st += 32;
  }
}

// faults of words [wi0, wi1) of group grp (row buffer B of the group, zeroed by the caller)
template <int G, bool OFF16, bool UNIFORM>
__device__ __forceinline__ void aff_group_faults(const DevProg& P, const AffTabs<OFF16>& T, uint32_t* B, uint64_t seed,
                                                 uint64_t word0, uint32_t grp, uint32_t W, int lane, uint32_t wi0,
                                                 uint32_t wi1) {
#if defined(FS_AFF_DIAG) && (FS_AFF_DIAG == 3 || FS_AFF_DIAG == 6)
  return;  // diagnostic: no fault pass
#endif
  if (P.num_runs == 1 && __ldg(P.run_len) > 0 && __ldg(P.run_len) < (1 << 20)) {
    AffRun1 R;
    R.start = __ldg(P.run_start);
    R.limit = 32u * __ldg(P.run_len);
    R.lp = __ldg(P.run_lp);
    R.q = __ldg(P.run_q);
    for (uint32_t wi = wi0; wi < wi1; wi++) {
      const uint32_t w = grp * G + wi;
      if (w >= W) break;
      aff_word_faults_1run<OFF16, UNIFORM>(T, B, wi, seed, word0 + w, lane, R);
    }
  } else {
    for (uint32_t wi = wi0; wi < wi1; wi++) {
      const uint32_t w = grp * G + wi;
      if (w >= W) break;
      aff_word_faults<OFF16, UNIFORM>(P, T, B, wi, seed, word0 + w, lane);
    }
  }
}

// barrier of the two warps of pair `id` (named barriers 0..15; barrier 0 serves the block-wide
// __syncthreads of the table load only before any pair uses it)
__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

}  // namespace fs
