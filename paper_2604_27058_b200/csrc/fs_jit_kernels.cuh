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

// word-level flattened hazard process of philox_noise_word(), XORing into physical slots:
// pslot[j] = physical frame slot of Pauli entry j under the renaming at this block.
__device__ __noinline__ void jit_noise_block(const DevProg& P, uint32_t* F, const uint16_t* __restrict__ pslot,
                                             uint64_t seed, uint64_t word, int instr, int plan_off, int plan_cnt) {
  const double* S = P.cum_hazard;
  PhiloxStream ps;
  ps.init(seed, word, (uint32_t)instr, TAG_NOISE);
  for (int pi = 0; pi < plan_cnt; pi++) {
    const int a = __ldg(P.plans + 2 * (plan_off + pi)), b = __ldg(P.plans + 2 * (plan_off + pi) + 1);
    if (a < 0) {
      const int site = b, nc = num_cases(P, site);
      for (int l = 0; l < 32; l++) {
        int c = __ldg(P.site_case_off + site);
        if (nc > 1) c = pick_case(P, site, ps.uniform());
        const int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
        for (int j = off; j < end; j++) F[(uint32_t)__ldg(pslot + j) * 32] ^= 1u << l;
      }
      continue;
    }
    const double Sa = __ldg(S + a);
    const double H = __dsub_rn(__ldg(S + b), Sa);
    if (!(H > 0.0)) continue;
    const double total = __dmul_rn(32.0, H);
    double t = 0.0;
    for (;;) {
      t = __dadd_rn(t, -log1p(-ps.uniform()));
      if (!(t < total)) break;
      const int l = (int)__ddiv_rn(t, H);
      if (l > 31) break;
      const double local = __dadd_rn(Sa, __dsub_rn(t, __dmul_rn((double)l, H)));
      const int idx = bisect_right(S, local, a + 1, b + 1);
      if (idx > b) { t = __dmul_rn((double)(l + 1), H); continue; }
      const int site = idx - 1;
      int c = __ldg(P.site_case_off + site);
      if (num_cases(P, site) > 1) c = pick_case(P, site, ps.uniform());
      const int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
      for (int j = off; j < end; j++) F[(uint32_t)__ldg(pslot + j) * 32] ^= 1u << l;
      t = __dadd_rn(__dmul_rn((double)l, H), __dsub_rn(__ldg(S + site + 1), Sa));
    }
  }
}

__device__ __forceinline__ uint4 coin_block(uint64_t seed, uint64_t wabs, int blk) {
  return philox((uint32_t)wabs, (uint32_t)(wabs >> 32), (uint32_t)blk, TAG_COIN << 24, seed);
}

}  // namespace fs
