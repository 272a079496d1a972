// fs_device.cuh -- device-side program view, random streams and small helpers shared by the
// sm_100a engines.  See DESIGN.md for the data layout and stream definitions.
#pragma once
#ifdef __CUDACC_RTC__  // NVRTC (program-specialised kernels, fs_jit.cuh): no host headers
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef unsigned char uint8_t;
typedef signed char int8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef unsigned long long uintptr_t;
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

#include "../../include/fs_sampler.h"
#include "fs_lntab.h"

namespace fs {

constexpr double kInvSqrt2 = 0.70710678118654757;  // 1/math.sqrt(2.0), runtime.py:46
constexpr double kBranchFloor = 1e-12;               // runtime.py:47
constexpr int kSmall = 8;                            // runtime.py:48 (selects the reduction formula)
constexpr uint32_t kFull = 0xFFFFFFFFu;

// Device copy of the serialized program (include/fs_sampler.h).  All tables live in one
// device allocation; the struct is passed by value as a kernel parameter.
struct DevProg {
  int n, k_max, num_instrs, R, U, D, O, E, num_slots, has_psel;
  const int* __restrict__ instrs;  // [N][8]
  const int* __restrict__ schedule;
  const double* __restrict__ fparams;
  const uint32_t* __restrict__ gates;
  const uint32_t* __restrict__ paulis;
  const int* __restrict__ reclists;
  const double* __restrict__ site_prob;
  const int* __restrict__ site_case_off;
  const double* __restrict__ case_cum;
  const int* __restrict__ case_pauli_off;
  const double* __restrict__ cum_hazard;
  const int* __restrict__ plans;
  const int* __restrict__ record_out;
  const int* __restrict__ bit_slot;
  // Philox noise runs (host-computed): maximal runs of consecutive sites with equal 0<p<1
  // (run_len > 0, run_lp = 1/log1p(-q), run_q = q = the run's largest p) or a single certain
  // site (run_len == 0)
  int num_runs;
  const int* __restrict__ run_start;
  const int* __restrict__ run_len;
  const double* __restrict__ run_lp;
  const double* __restrict__ run_q;
  const int* __restrict__ next_array;   // [N] first array instruction >= i (N if none); with frame
                                        // matrices also the first FrameGates instruction
  // FrameGates as GF(2) matrices (block engine, 2n <= 128): instruction i maps the frame vector
  // v = (x_0..x_{n-1}, z_0..z_{n-1}) to v' with v'_r = parity(row_r & v); rows are 4 words
  const uint32_t* __restrict__ frame_mat;
  const int* __restrict__ frame_mat_off;  // [N] word offset of instruction i's rows, -1 if none
  // star groups (block engine, fs_sampler.cu fs_program_create): fuse_at[i] = group starting at
  // ArrayGate i or -1; fuse = 8-word descriptors
  const int* __restrict__ fuse_at;
  const int* __restrict__ fuse;
  // per-case frame masks, 4 words each (x_q at bit q, z_q at bit n + q); NULL when 2n > 128
  const uint4* __restrict__ case_mask;
};

struct RunArgs {
  uint64_t seed, shot0, nshots;
  uint32_t flags;
  uint32_t W;          // output words = ceil(nshots/32)
  uint32_t ostride;    // row stride of the output words (== W except for chunked launches)
  uint32_t* meas;      // [U][W]
  uint32_t* det;       // [D][W]
  uint32_t* obs;       // [O][W]
  uint32_t* accepted;  // [W]
  uint32_t* error;     // [W]
  int* status;         // max FS_ERR_SHOT_* seen
  int prezeroed;       // outputs memset to 0 => a warp whose shots all halted may stop early
  // trace mode
  const int16_t* fault_modes;  // [nshots][E]
  const int8_t* forced;        // [nshots][R]
  int stop;                    // instructions to execute
  uint8_t* t_fx;
  uint8_t* t_fz;
  double* t_gamma;
  double* t_amps;
  uint32_t* t_draws;
  uint8_t* t_rec;       // [nshots][R] every record bit (trace)
  // checkpoints (trace): state after instructions [0, cp_at[j]) for j < ncp
  int ncp;
  const int* cp_at;          // device [ncp], ascending
  const uint64_t* cp_off;    // device [ncp]: offset (complex elements) of checkpoint j's amplitude block
  uint8_t* cp_valid;         // [ncp][nshots]
  uint8_t* cp_fx;            // [ncp][nshots][n]
  uint8_t* cp_fz;
  double* cp_gamma;          // [ncp][nshots][2]
  double* cp_amps;           // blocks [nshots][2^k_j][2] at cp_off[j]
  const uint32_t* draw0;  // [nshots] reference-stream draws consumed before the program
                          // (stratified sampling: StratumSpec.draw_forced), NULL = 0
  // general engine: per-resident-warp array storage when it does not fit in shared memory
  double2* scratch;
  int arr_log2;  // log2 capacity (k_max)
};

// ------------------------------------------------------------------ random streams
enum : uint32_t { TAG_COIN = 1, TAG_BORN = 2, TAG_NOISE = 3, TAG_FORCED = 4, TAG_STRATUM = 5 };

__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c1 = lo1;
    c3 = lo0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// coin word of MeasDormantRandom number `ord` for 32-shot word `wabs`: 4 coin words per block
__device__ __forceinline__ uint32_t coin_word(uint64_t seed, uint64_t wabs, int ord) {
  const uint4 b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), (uint32_t)(ord >> 2), TAG_COIN << 24, seed);
  const int j = ord & 3;
  return j == 0 ? b.x : (j == 1 ? b.y : (j == 2 ? b.z : b.w));
}

__device__ __forceinline__ double u64_to_unit(uint64_t x) {
  return __dmul_rn(__ull2double_rn(x), 5.421010862427522e-20);
}

// ln(U) for the noise stream's gap draws, U = (2 * (bits >> 12) + 1) * 2^-53 in (0, 1) (exact).
// U = m * 2^e with m in [1, 2) read off the bits; ln m = T_k + ln(1 + r) with the 64-interval
// table of fs_lntab.h (r = fma(m, inv_k, -1), |r| < 2^-7) and an 8-term series for ln(1 + r).
// IEEE basic operations and explicit FMAs only, in a fixed order, so the CPU oracle
// (oracle/fs_oracle.c ln_unit) reproduces it bit for bit; |error| <= 1e-14 absolute.
__device__ const double2 kLnTab[FS_LN_TAB_ENTRIES] = FS_LN_TAB_INIT;

__device__ __forceinline__ double ln_unit_t(uint64_t bits, const double2* __restrict__ tab) {
  const uint64_t v = ((bits >> 12) << 1) | 1ull;
  const int p = 63 - __clzll((long long)v);
  const uint64_t mant = (v << (52 - p)) & ((1ull << 52) - 1ull);
  const double m = __longlong_as_double((long long)((1023ull << 52) | mant));
  const double2 t = tab[mant >> 46];
  const double r = fma(m, t.x, -1.0);
  double P = -0.125;
  P = fma(P, r, 0x1.2492492492492p-3);
  P = fma(P, r, -0x1.5555555555555p-3);
  P = fma(P, r, 0x1.999999999999ap-3);
  P = fma(P, r, -0.25);
  P = fma(P, r, 0x1.5555555555555p-2);
  P = fma(P, r, -0.5);
  P = fma(P, r, 1.0);
  P = __dmul_rn(P, r);
  return __dadd_rn(__dadd_rn(__dmul_rn((double)(p - 53), 0x1.62e42fefa39efp-1), t.y), P);
}
__device__ __forceinline__ double ln_unit(uint64_t bits) { return ln_unit_t(bits, kLnTab); }

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// reference ShotRng (rng.py:24-71): key = mix(mix(seed) ^ shot); draw c = mix(key + c*golden)
struct SplitMix {
  uint64_t key;
  uint32_t count;
  __device__ __forceinline__ void reset(uint64_t seed, uint64_t shot) {
    key = mix64(mix64(seed) ^ shot);
    count = 0;
  }
  __device__ __forceinline__ uint64_t next() {
    uint64_t c = count++;
    return mix64(key + c * 0x9E3779B97F4A7C15ULL);
  }
  __device__ __forceinline__ double uniform() { return u64_to_unit(next()); }
  __device__ __forceinline__ int bit() { return (int)(next() >> 63); }
};

// per-(shot|word, instruction, tag) Philox stream: draw j uses block j/2, half j%2
struct PhiloxStream {
  uint64_t seed, ctr;
  uint32_t instr, tag, j;
  uint4 blk;
  __device__ __forceinline__ void init(uint64_t s, uint64_t c, uint32_t i, uint32_t t) {
    seed = s; ctr = c; instr = i; tag = t; j = 0;
  }
  __device__ __forceinline__ uint64_t next() {
    if ((j & 1) == 0) blk = philox((uint32_t)ctr, (uint32_t)(ctr >> 32), instr, (tag << 24) | (j >> 1), seed);
    uint64_t r = (j & 1) ? (((uint64_t)blk.w << 32) | blk.z) : (((uint64_t)blk.y << 32) | blk.x);
    j++;
    return r;
  }
  __device__ __forceinline__ double uniform() { return u64_to_unit(next()); }
};

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// fused variant for the program-specialised kernels (records unchanged; amplitudes differ from the
// reference only in the last ulp, within the 1e-10 parity tolerance)
__device__ __forceinline__ double2 cmul_f(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}
// cmul_f(u, a) for a u with a zero imaginary (cmul_re) or real (cmul_im) part: the vanishing
// products drop out of the FMAs exactly, so these give the same doubles with two multiplies
__device__ __forceinline__ double2 cmul_re(double ux, double2 a) { return make_double2(__dmul_rn(ux, a.x), __dmul_rn(ux, a.y)); }
__device__ __forceinline__ double2 cmul_im(double uy, double2 a) { return make_double2(-__dmul_rn(uy, a.y), __dmul_rn(uy, a.x)); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
// python complex * float (runtime.py: `buf[i] * scale`): real-scaled, no FMA contraction
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(__dmul_rn(a.x, s), __dmul_rn(a.y, s)); }
__device__ __forceinline__ double cnorm2(double2 a) { return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)); }

// insert a 0 bit at position a (Retire / MeasCollapse gather, backend.py:436-441)
__device__ __forceinline__ uint32_t ins0(uint32_t i, int a) {
  uint32_t lowmask = (1u << a) - 1u;
  return ((i & ~lowmask) << 1) | (i & lowmask);
}

__device__ __forceinline__ uint64_t ins0_64(uint64_t i, int a) {
  const uint64_t lowmask = (1ull << a) - 1ull;
  return ((i & ~lowmask) << 1) | (i & lowmask);
}

// ------------------------------------------------------------------ noise helpers
__device__ __forceinline__ int bisect_right(const double* __restrict__ S, double x, int lo, int hi) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (x < __ldg(S + mid)) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// _pick_case (runtime.py:702-707) with a supplied uniform
__device__ __forceinline__ int pick_case(const DevProg& P, int site, double u) {
  int c0 = __ldg(P.site_case_off + site), nc = __ldg(P.site_case_off + site + 1) - c0;
  double x = u * __ldg(P.site_prob + site);
  int c = bisect_right(P.case_cum + c0, x, 0, nc);
  return c0 + (c < nc - 1 ? c : nc - 1);
}

// case of a fault given x uniform on [0, p_site): bisect_right over the site's cumulative case
// probabilities, clamped to the last case (the _pick_case law, runtime.py:702-707)
__device__ __forceinline__ int pick_case_x(const DevProg& P, int site, double x) {
  int c0 = __ldg(P.site_case_off + site), nc = __ldg(P.site_case_off + site + 1) - c0;
  int c = bisect_right(P.case_cum + c0, x, 0, nc);
  return c0 + (c < nc - 1 ? c : nc - 1);
}

__device__ __forceinline__ int num_cases(const DevProg& P, int site) {
  return __ldg(P.site_case_off + site + 1) - __ldg(P.site_case_off + site);
}

}  // namespace fs
