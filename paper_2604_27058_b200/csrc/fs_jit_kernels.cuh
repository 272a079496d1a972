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

__device__ __forceinline__ uint4 coin_block(uint64_t seed, uint64_t wabs, int blk) {
  return philox((uint32_t)wabs, (uint32_t)(wabs >> 32), (uint32_t)blk, TAG_COIN << 24, seed);
}

}  // namespace fs
