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
