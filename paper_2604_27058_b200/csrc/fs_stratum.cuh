// fs_stratum.cuh -- stratified importance sampling (runtime.py:886-945) on the device.
//
// StratumSpec(prog, w) conditions every shot on exactly w realised faults.  Its draw_forced
// (runtime.py:915-932) walks the sites in order with the suffix Poisson-binomial table
//   T[i][m] = Pr[m faults among sites i..E-1]   (host-built, fs_sampler.cu stratum_table)
// and forces site i with probability p_i * T[i+1][need-1] / T[i][need], until `need` faults are
// placed (or the remaining sites must all fire).  One thread per shot writes the shot's forced
// fault modes (1 = trigger, case drawn by the program; 2 = skip) into the dense [n][E] trace
// input consumed by the forced-fault path of every engine, plus the number of reference-stream
// draws it consumed: the program's own draws continue from there (the reference uses one
// ShotRng for both).  Engine stream: the uniforms come from Philox blocks
// (shot, 0xFFFFFFFF, TAG_STRATUM << 24 | t / 2), two 64-bit draws per block.
#pragma once
#include "fs_device.cuh"

namespace fs {

__global__ void fill_modes_kernel(int16_t* __restrict__ modes, uint64_t count) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t n8 = count / 8;
  if (i < n8) {
    reinterpret_cast<uint4*>(modes)[i] = make_uint4(0x00020002u, 0x00020002u, 0x00020002u, 0x00020002u);
  } else if (i == n8) {
    for (uint64_t j = n8 * 8; j < count; j++) modes[j] = 2;
  }
}

template <bool SPLITMIX>
__global__ void __launch_bounds__(128) stratum_kernel(DevProg P, const double* __restrict__ T, int w,
                                                      uint64_t seed, uint64_t shot0, uint64_t n,
                                                      int16_t* __restrict__ modes, uint32_t* __restrict__ draw0) {
  const uint64_t si = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (si >= n) return;
  const uint64_t shot = shot0 + si;
  const int E = P.E, w1 = w + 1;
  int16_t* m = modes + si * (size_t)E;
  SplitMix sm;
  if (SPLITMIX) sm.reset(seed, shot);
  uint32_t t = 0;  // engine-stream draw index
  uint4 blk = make_uint4(0, 0, 0, 0);
  int need = w;
  for (int i = 0; i < E && need > 0; i++) {
    const int remaining = E - i;
    if (remaining == need) {
      for (int j = i; j < E; j++) m[j] = 1;
      break;
    }
    const double p_here = __dmul_rn(__ldg(P.site_prob + i), __ldg(T + (size_t)(i + 1) * w1 + (need - 1)));
    const double p_total = __ldg(T + (size_t)i * w1 + need);
    double u;
    if (SPLITMIX) {
      u = sm.uniform();
    } else {
      if (!(t & 1)) blk = philox((uint32_t)shot, (uint32_t)(shot >> 32), 0xFFFFFFFFu, (TAG_STRATUM << 24) | (t >> 1), seed);
      u = u64_to_unit((t & 1) ? (((uint64_t)blk.w << 32) | blk.z) : (((uint64_t)blk.y << 32) | blk.x));
      t++;
    }
    if (__dmul_rn(u, p_total) < p_here) {
      m[i] = 1;
      need--;
    }
  }
  if (draw0) draw0[si] = SPLITMIX ? sm.count : 0u;
}

}  // namespace fs
