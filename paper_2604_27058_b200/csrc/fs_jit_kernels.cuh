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

// Pre-expanded noise flips for the specialised frame kernel.  noise_flip_kernel generates the
// word's faults (WordFaultGen, the engine stream) and expands every fault into its frame flips
// (physical slot under the renaming at its NoiseBlock, lane bit): flips[i][W] = slot << 5 | lane,
// grouped by NoiseBlock with bcount[b][W] flips per block.  bcount[0][w] == ~0 marks a word whose
// flips overflowed `cap`; the frame kernel then regenerates that word's stream in place.
__global__ void __launch_bounds__(256) noise_flip_kernel(DevProg P, uint64_t seed, uint64_t word0, uint32_t W,
                                                        const uint16_t* __restrict__ pslot,
                                                        const int* __restrict__ site_block, int nblocks,
                                                        uint32_t* __restrict__ flips, uint32_t* __restrict__ bcount,
                                                        uint32_t cap) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
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
    while (blk < b) {  // close the blocks before this fault's block
      bcount[(size_t)blk * W + w] = nb;
      nb = 0;
      blk++;
    }
    const int off = __ldg(P.case_pauli_off + cs), end = __ldg(P.case_pauli_off + cs + 1);
    if (n + (uint32_t)(end - off) > cap) { over = true; break; }
    for (int j = off; j < end; j++) flips[(size_t)(n++) * W + w] = ((uint32_t)__ldg(pslot + j) << 5) | (uint32_t)lane;
    nb += (uint32_t)(end - off);
  }
  if (over) {
    bcount[w] = 0xFFFFFFFFu;
    return;
  }
  for (; blk < nblocks; blk++) {
    bcount[(size_t)blk * W + w] = nb;
    nb = 0;
  }
}

// apply the n flips of this word's current NoiseBlock
__device__ __forceinline__ void jit_apply_flips(uint32_t* F, const uint32_t* __restrict__ flips, uint32_t W,
                                                uint32_t w, uint32_t& cur, uint32_t n) {
  uint32_t t = 0;
  for (; t + 4 <= n; t += 4) {
    const uint32_t e0 = __ldg(flips + (size_t)(cur + t) * W + w), e1 = __ldg(flips + (size_t)(cur + t + 1) * W + w);
    const uint32_t e2 = __ldg(flips + (size_t)(cur + t + 2) * W + w), e3 = __ldg(flips + (size_t)(cur + t + 3) * W + w);
    F[(e0 >> 5) * 32] ^= 1u << (e0 & 31);
    F[(e1 >> 5) * 32] ^= 1u << (e1 & 31);
    F[(e2 >> 5) * 32] ^= 1u << (e2 & 31);
    F[(e3 >> 5) * 32] ^= 1u << (e3 & 31);
  }
  for (; t < n; t++) {
    const uint32_t e = __ldg(flips + (size_t)(cur + t) * W + w);
    F[(e >> 5) * 32] ^= 1u << (e & 31);
  }
  cur += n;
}

__device__ __forceinline__ uint4 coin_block(uint64_t seed, uint64_t wabs, int blk) {
  return philox((uint32_t)wabs, (uint32_t)(wabs >> 32), (uint32_t)blk, TAG_COIN << 24, seed);
}

}  // namespace fs
