// fs_hbm_fused.cuh -- fused tile passes of the large-k engine.
//
// A pass applies a run of array instructions (H, S, S_DAG, CX, CZ, ArrayRot, Expand) to every
// shot's HBM-resident array in ONE read + write of the array.  The host planner (fs_sampler.cu
// plan_hbm) chooses per pass a set T of kTileBits physical axes that contains every axis an
// instruction mixes along (H: its axis, CX: its target, Expand: the new axis); diagonal
// instructions (CZ, S, ArrayRot) and CX controls read their bits from the element index, so they
// may use any axis.  A CTA loads a tile = the 2^kTileBits amplitudes that differ only in T
// (the other live axes are fixed by the tile index, dead axes are 0) into shared memory, applies
// the pass's instructions there and writes the tile back.  The low physical axes 0..2 are always
// in T (consecutive threads then touch 128-byte runs).  Consecutive diagonal instructions are
// applied in one register sweep.
#pragma once
#include "fs_hbm.cuh"

namespace fs {

constexpr int kTileBits = 12;   // 4096 amplitudes = 64 KiB of shared memory per tile
constexpr int kTileThreads = 256;
constexpr int kTileElems = (1 << kTileBits) / kTileThreads;  // 16 per thread

enum TileOpKind : int8_t { TO_H = 0, TO_S, TO_SDAG, TO_CX, TO_CZ, TO_ROT, TO_EXPAND };

struct TileOp {
  int8_t kind;
  int8_t la, lb;  // local (tile) bit of the op's axes, -1 when the axis is outside the tile
  int8_t pa, pb;  // physical axes (for bits taken from the tile base)
  int8_t diag_run;  // number of consecutive diagonal ops starting here (0 if not diagonal)
  int16_t pad;
  int instr;      // parity row (ArrayRot / Expand)
  double2 c0, c1, c2, c3;
};

struct PassDesc {
  int nops, op_off;
  int nbase;
  int ncode, code_off;    // microcode words (see below)
  int nconst, const_off;  // PassConst entries
  int8_t T[kTileBits];   // physical axis of each tile bit
  int8_t base[32];       // live physical axes outside the tile (tile index bits)
  uint32_t dep_hi[kTileElems];  // physical offset of element j = tid + 256 * j, high part
  int8_t Tf[kTileBits];          // layout at the end of the pass (after register swaps)
  uint32_t dep_hi_f[kTileElems];
};

__device__ __forceinline__ uint64_t deposit_bits(uint64_t v, const int8_t* pos, int n) {
  uint64_t g = 0;
  for (int i = 0; i < n; i++) g |= ((v >> i) & 1ull) << pos[i];
  return g;
}

// bit of physical axis `p` (tile-local position `l`) for local index `li` in the tile at `base`
__device__ __forceinline__ int axis_bit(int l, int p, uint32_t li, uint64_t base) {
  return l >= 0 ? (int)((li >> l) & 1u) : (int)((base >> p) & 1ull);
}

// ---- register-blocked tile: thread t holds elements l = t + 256 j (j = 0..15), i.e. tile bits
// 0..7 are "thread bits" (exchanged through shared memory) and bits 8..11 "register bits"
template <int R>
__device__ __forceinline__ void reg_h(double2 (&v)[kTileElems]) {
#pragma unroll
  for (int j = 0; j < kTileElems; j++)
    if (!((j >> R) & 1)) {
      const double2 lo = v[j], hi = v[j | (1 << R)];
      v[j] = cscale(cadd(lo, hi), kInvSqrt2);
      v[j | (1 << R)] = cscale(csub(lo, hi), kInvSqrt2);
    }
}
template <int R>
__device__ __forceinline__ void reg_cx(double2 (&v)[kTileElems], int ctl_kind, int ctl, uint32_t tid, uint64_t base) {
  // ctl_kind: 0 register bit ctl, 1 thread bit ctl, 2 base bit ctl (physical), 3 always
#pragma unroll
  for (int j = 0; j < kTileElems; j++)
    if (!((j >> R) & 1)) {
      const int cb = ctl_kind == 0 ? (j >> ctl) & 1 : ctl_kind == 1 ? (int)((tid >> ctl) & 1u)
                   : ctl_kind == 2 ? (int)((base >> ctl) & 1ull) : 1;
      if (cb) {
        const double2 t0 = v[j];
        v[j] = v[j | (1 << R)];
        v[j | (1 << R)] = t0;
      }
    }
}
template <int R>
__device__ __forceinline__ void reg_expand(double2 (&v)[kTileElems], double2 ph0, double2 ph1) {
#pragma unroll
  for (int j = 0; j < kTileElems; j++)
    if (!((j >> R) & 1)) {
      const double2 s = v[j];
      v[j] = cmul(s, ph0);
      v[j | (1 << R)] = cmul(s, ph1);
    }
}

// ---- pass microcode (host-compiled by plan_hbm, shot-independent)
// Positions are bits of the extended local index X = tid | j << 8 | tile << 12: tile bits 0..7 are
// thread bits, 8..11 register bits (element j of the thread), then the pass's base axes.
//   MC_H   | m << 4                      Hadamard along tile bit m
//   MC_CX  | m << 4 | c << 9             X on tile bit m controlled by position c
//   MC_EXP | m << 4 | k << 16            Expand onto tile bit m, constants k
// Register bits (m >= 8) are updated in registers; a lane bit (m < 5) exchanges with the partner
// lane by register shuffles; a warp bit (5 <= m < 8) exchanges the tile through shared memory.
//   MC_DIAG| nterm << 4 | nrot << 12, then lin0, lin1, M0..M3, sR | QQ << 16,
//            nterm x (a, N_a), nrot x (a | k << 8)
// A diagonal run (CZ / S / S_DAG / ROT, which commute) multiplies element X by
// i^P(X) * prod_rot c(X) with the Z4 quadratic form
//   P(X) = sum_a s_a x_a + 2 sum_{CZ(a,b)} x_a x_b.
// Over the constant bits (thread + tile index) of a thread it evaluates to
//   e0 = popc(X & lin0) + 2 popc(X & lin1) + 2 sum_a x_a popc(X & N_a),
//   e_R = s_R + 2 popc(X & M_R)          (coefficient of register bit R),
// plus 2 * QQ (the register-register CZ pattern over j), so a run costs a few popcounts per
// thread instead of one update of every element per instruction.
enum : uint32_t { MC_H = 0, MC_CX = 1, MC_EXP = 2, MC_DIAG = 3 };

struct PassConst {  // ROT: c0 / c1 = factor of bit 0 / 1; EXPAND: c0..c3 (parity 0: c0, c1; 1: c2, c3)
  double2 c0, c1, c2, c3;
  int instr, kind, pad0, pad1;
};
constexpr int kPassMaxOps = kTileThreads;  // tile ops per pass (bounds constants and microcode)
constexpr int kPassMaxCode = 2048;
constexpr int kPassSmem = (16 << kTileBits) + 4 * kPassMaxCode + 32 * kPassMaxOps;

__device__ __forceinline__ uint32_t reg_mask(int R) {  // j in [0,16) with bit R set
  return (uint32_t)((0xFF00F0F0CCCCAAAAull >> (16 * R)) & 0xFFFFu);
}

__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

// i^P(j) from the run's coefficients: e0 on every element, eR[R] on elements with bit R of j,
// 2 * QQ (register-register CZ pattern over j); P held as two 16-bit planes (bit 0 / bit 1)
__device__ __forceinline__ void ipow_planes(uint32_t e0, const uint32_t (&eR)[4], uint32_t QQ, uint32_t& Lm,
                                            uint32_t& Hm) {
  Lm = (e0 & 1u) ? 0xFFFFu : 0u;
  Hm = (e0 & 2u) ? 0xFFFFu : 0u;
#pragma unroll
  for (int R = 0; R < 4; R++) {
    const uint32_t m = reg_mask(R);
    if (eR[R] & 1u) {
      const uint32_t cy = Lm & m;
      Lm ^= m;
      Hm ^= cy;
    }
    if (eR[R] & 2u) Hm ^= m;
  }
  Hm ^= QQ;
}

__device__ __forceinline__ void apply_ipow(double2 (&v)[kTileElems], uint32_t Lm, uint32_t Hm) {
  if (!(Lm | Hm)) return;
#pragma unroll
  for (int j = 0; j < kTileElems; j++) {
    const uint32_t lb = (Lm >> j) & 1u, hb = (Hm >> j) & 1u;
    double x = v[j].x, y = v[j].y;
    if (lb) { const double t = x; x = y; y = t; }
    if (lb ^ hb) x = -x;
    if (hb) y = -y;
    v[j] = make_double2(x, y);
  }
}

// v[j] *= g * prod_{R : bit R of j, R in rreg} d[R]
__device__ __forceinline__ void apply_rot(double2 (&v)[kTileElems], double2 g, const double2 (&d)[4], uint32_t rreg) {
  if (rreg) {
    double2 t01[4];
    t01[0] = g;
    t01[1] = cmul(g, d[0]);
    t01[2] = cmul(g, d[1]);
    t01[3] = cmul(t01[1], d[1]);
    const double2 d23 = cmul(d[2], d[3]);
#pragma unroll
    for (int j = 0; j < kTileElems; j++) {
      const int hi = j >> 2;
      const double2 f = hi == 0 ? t01[j & 3] : cmul(t01[j & 3], hi == 1 ? d[2] : hi == 2 ? d[3] : d23);
      v[j] = cmul(v[j], f);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kTileElems; j++) v[j] = cmul(v[j], g);
  }
}

__device__ __forceinline__ void diag_run_apply(double2 (&v)[kTileElems], const uint32_t* __restrict__ c,
                                               const double2* __restrict__ cs, uint32_t X0) {
  const uint32_t w = c[0];
  const int nterm = (w >> 4) & 0xFF, nrot = (w >> 12) & 0xFF;
  uint32_t e0 = __popc(X0 & c[1]) + 2u * __popc(X0 & c[2]);
  uint32_t q = 0;
  for (int t = 0; t < nterm; t++) {
    const uint32_t a = c[8 + 2 * t], na = c[9 + 2 * t];
    q += ((X0 >> a) & 1u) * __popc(X0 & na);
  }
  e0 += 2u * q;
  const uint32_t sr = c[7];
  uint32_t eR[4];
#pragma unroll
  for (int R = 0; R < 4; R++) eR[R] = ((sr >> (2 * R)) & 3u) + 2u * __popc(X0 & c[3 + R]);
  uint32_t Lm, Hm;
  ipow_planes(e0, eR, sr >> 16, Lm, Hm);
  apply_ipow(v, Lm, Hm);
  if (nrot == 0) return;
  const uint32_t* rt = c + 8 + 2 * nterm;
  uint32_t rreg = 0;
  double2 g = make_double2(1, 0);
  double2 d[4];
#pragma unroll
  for (int q4 = 0; q4 < 4; q4++) d[q4] = make_double2(1, 0);
  for (int r = 0; r < nrot; r++) {
    const uint32_t rw = rt[r];
    const int xa = rw & 31, k = rw >> 8;
    const double2 ca = cs[2 * k], cb = cs[2 * k + 1];
    if ((unsigned)(xa - 8) < 4u) {
      const int R = xa - 8;
      g = cmul(g, ca);
      const double2 rat = cdiv(cb, ca);
#pragma unroll
      for (int q4 = 0; q4 < 4; q4++)
        if (q4 == R) d[q4] = cmul(d[q4], rat);
      rreg |= 1u << R;
    } else {
      g = cmul(g, ((X0 >> xa) & 1u) ? cb : ca);
    }
  }
  apply_rot(v, g, d, rreg);
}

// ---- thread-bit exchanges (shared by the interpreter and the generated pass kernels) --------
// control mask over j of a CX whose control sits at extended position xa
__device__ __forceinline__ uint32_t cx_ctl_mask(int xa, uint32_t X0) {
  return (unsigned)(xa - 8) < 4u ? reg_mask(xa - 8) : (((X0 >> xa) & 1u) ? 0xFFFFu : 0u);
}
// lane bit m < 5: partner lane by register shuffles.  H: bit 0 -> (v + p)/sqrt2, bit 1 -> (p - v)/sqrt2
__device__ __forceinline__ void xlane_h(double2 (&v)[kTileElems], uint32_t tid, int m) {
  const double sg = ((tid >> m) & 1u) ? -1.0 : 1.0;
#pragma unroll
  for (int j = 0; j < kTileElems; j++) {
    const double px = __shfl_xor_sync(0xFFFFFFFFu, v[j].x, 1 << m), py = __shfl_xor_sync(0xFFFFFFFFu, v[j].y, 1 << m);
    v[j] = make_double2(__dmul_rn(__fma_rn(sg, v[j].x, px), kInvSqrt2), __dmul_rn(__fma_rn(sg, v[j].y, py), kInvSqrt2));
  }
}
__device__ __forceinline__ void xlane_cx(double2 (&v)[kTileElems], int m, uint32_t cm) {
#pragma unroll
  for (int j = 0; j < kTileElems; j++) {
    const double px = __shfl_xor_sync(0xFFFFFFFFu, v[j].x, 1 << m), py = __shfl_xor_sync(0xFFFFFFFFu, v[j].y, 1 << m);
    if ((cm >> j) & 1u) v[j] = make_double2(px, py);
  }
}
// expand: the bit-1 half gets the bit-0 partner times ph1, the bit-0 half is scaled by ph0
__device__ __forceinline__ void xlane_exp(double2 (&v)[kTileElems], uint32_t tid, int m, double2 ph0, double2 ph1) {
  const bool mb = (tid >> m) & 1u;
  const double2 ph = mb ? ph1 : ph0;
#pragma unroll
  for (int j = 0; j < kTileElems; j++) {
    const double px = __shfl_xor_sync(0xFFFFFFFFu, v[j].x, 1 << m), py = __shfl_xor_sync(0xFFFFFFFFu, v[j].y, 1 << m);
    v[j] = cmul(mb ? make_double2(px, py) : v[j], ph);
  }
}
// warp bit 5 <= m < 8: exchange the tile with thread tid ^ (1 << m) through shared memory
__device__ __forceinline__ void xsmem_h(double2 (&v)[kTileElems], double2* T, uint32_t tid, int m) {
#pragma unroll
  for (int j = 0; j < kTileElems; j++) T[tid + kTileThreads * j] = v[j];
  __syncthreads();
  const uint32_t pt = tid ^ (1u << m);
  const double sg = ((tid >> m) & 1u) ? -1.0 : 1.0;
#pragma unroll
  for (int j = 0; j < kTileElems; j++) {
    const double2 pv = T[pt + kTileThreads * j];
    v[j] = make_double2(__dmul_rn(__fma_rn(sg, v[j].x, pv.x), kInvSqrt2), __dmul_rn(__fma_rn(sg, v[j].y, pv.y), kInvSqrt2));
  }
  __syncthreads();
}
__device__ __forceinline__ void xsmem_cx(double2 (&v)[kTileElems], double2* T, uint32_t tid, int m, uint32_t cm) {
#pragma unroll
  for (int j = 0; j < kTileElems; j++) T[tid + kTileThreads * j] = v[j];
  __syncthreads();
  const uint32_t pt = tid ^ (1u << m);
#pragma unroll
  for (int j = 0; j < kTileElems; j++)
    if ((cm >> j) & 1u) v[j] = T[pt + kTileThreads * j];
  __syncthreads();
}
__device__ __forceinline__ void xsmem_exp(double2 (&v)[kTileElems], double2* T, uint32_t tid, int m, double2 ph0,
                                          double2 ph1) {
#pragma unroll
  for (int j = 0; j < kTileElems; j++) T[tid + kTileThreads * j] = v[j];
  __syncthreads();
  const uint32_t pt = tid ^ (1u << m);
  const bool mb = (tid >> m) & 1u;
  const double2 ph = mb ? ph1 : ph0;
#pragma unroll
  for (int j = 0; j < kTileElems; j++) {
    const double2 pv = T[pt + kTileThreads * j];
    v[j] = cmul(mb ? pv : v[j], ph);
  }
  __syncthreads();
}

// ---- half-buffer warp-bit exchanges (the specialised pass kernels keep a 64 KiB staging buffer
// for the next tile, so the exchange goes through 32 KiB in two rounds of 8 elements)
template <int OP>  // 0 = H, 1 = CX (mask cm), 2 = Expand (ph0, ph1)
__device__ __forceinline__ void xsmem_half(double2 (&v)[kTileElems], double2* T, uint32_t tid, int m, uint32_t cm,
                                           double2 ph0, double2 ph1) {
  const uint32_t pt = tid ^ (1u << m);
  const bool mb = (tid >> m) & 1u;
  const double sg = mb ? -1.0 : 1.0;
  const double2 ph = mb ? ph1 : ph0;
#pragma unroll
  for (int h = 0; h < 2; h++) {
#pragma unroll
    for (int j = 0; j < kTileElems / 2; j++) T[tid + kTileThreads * j] = v[8 * h + j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kTileElems / 2; j++) {
      const double2 pv = T[pt + kTileThreads * j];
      double2& x = v[8 * h + j];
      if (OP == 0) x = make_double2(__dmul_rn(__fma_rn(sg, x.x, pv.x), kInvSqrt2), __dmul_rn(__fma_rn(sg, x.y, pv.y), kInvSqrt2));
      else if (OP == 1) { if ((cm >> (8 * h + j)) & 1u) x = pv; }
      else x = cmul(mb ? pv : x, ph);
    }
    __syncthreads();
  }
}

// 16-byte asynchronous global -> shared copy (L2 only), and the wait for this thread's copies
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ---- TMA bulk copies (cp.async.bulk, completion counted in bytes on an mbarrier): the pass
// kernels stage a tile as 512 contiguous 128-byte runs (physical axes 0..2) instead of 4096 16-byte
// cp.async requests
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "FS_MBAR_WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra FS_MBAR_WAIT%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_addr(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

__global__ void __launch_bounds__(kTileThreads, 2) hbm_fused_pass_kernel(HbmState H, const PassDesc D,
                                                                        const uint32_t* __restrict__ code,
                                                                        const PassConst* __restrict__ consts,
                                                                        uint32_t W) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* T = reinterpret_cast<double2*>(smem_raw);
  uint32_t* mc = reinterpret_cast<uint32_t*>(smem_raw + (16 << kTileBits));
  double2* cs = reinterpret_cast<double2*>(smem_raw + (16 << kTileBits) + 4 * kPassMaxCode);
  const uint32_t shot = blockIdx.y;
  const uint32_t w = shot >> 5, bit = 1u << (shot & 31);
  if (!(H.alive[w] & bit)) return;
  const uint32_t tid = threadIdx.x;
  for (int i = tid; i < D.ncode; i += kTileThreads) mc[i] = code[D.code_off + i];
  for (int i = tid; i < D.nconst; i += kTileThreads) {  // resolve the shot's parities
    const PassConst& k = consts[D.const_off + i];
    const bool par = (H.par[(size_t)k.instr * W + w] & bit) != 0;
    double2 a = k.c0, b = k.c1;
    if (par) {
      if (k.kind == TO_ROT) { a = k.c1; b = k.c0; }
      else { a = k.c2; b = k.c3; }
    }
    cs[2 * i] = a;
    cs[2 * i + 1] = b;
  }
  uint32_t dep_lo = 0, dep_lo_f = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    dep_lo |= ((tid >> i) & 1u) << D.T[i];
    dep_lo_f |= ((tid >> i) & 1u) << D.Tf[i];
  }
  const uint64_t ntiles = 1ull << D.nbase;
  double2* __restrict__ A = H.amps + (size_t)shot * H.cap;
  const int ncode = D.ncode;
  __syncthreads();
  double2 v[kTileElems];
  for (uint64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const uint64_t base = deposit_bits(ti, D.base, D.nbase);
    const uint32_t X0 = tid | (uint32_t)(ti << kTileBits);
#pragma unroll
    for (int j = 0; j < kTileElems; j++) v[j] = A[base | dep_lo | D.dep_hi[j]];
    for (int pc = 0; pc < ncode;) {
      const uint32_t ow = mc[pc];
      const uint32_t kind = ow & 15u;
      if (kind == MC_DIAG) {
        diag_run_apply(v, mc + pc, cs, X0);
        pc += 8 + 2 * ((ow >> 4) & 0xFF) + ((ow >> 12) & 0xFF);
        continue;
      }
      pc++;
      const int m = (ow >> 4) & 15;
      if (m >= 8) {  // register bit: no data exchange
        const int R = m - 8;
        if (kind == MC_H) {
          if (R == 0) reg_h<0>(v); else if (R == 1) reg_h<1>(v); else if (R == 2) reg_h<2>(v); else reg_h<3>(v);
        } else if (kind == MC_CX) {
          const int xa = (ow >> 9) & 31;
          const bool creg = (unsigned)(xa - 8) < 4u;
          const int c = creg ? xa - 8 : (int)((X0 >> xa) & 1u);
          if (!creg && !c) continue;
          const int ck = creg ? 0 : 3;
          if (R == 0) reg_cx<0>(v, ck, c, tid, 0); else if (R == 1) reg_cx<1>(v, ck, c, tid, 0);
          else if (R == 2) reg_cx<2>(v, ck, c, tid, 0); else reg_cx<3>(v, ck, c, tid, 0);
        } else {  // MC_EXP
          const int k = ow >> 16;
          const double2 ph0 = cs[2 * k], ph1 = cs[2 * k + 1];
          if (R == 0) reg_expand<0>(v, ph0, ph1); else if (R == 1) reg_expand<1>(v, ph0, ph1);
          else if (R == 2) reg_expand<2>(v, ph0, ph1); else reg_expand<3>(v, ph0, ph1);
        }
        continue;
      }
      const uint32_t cm = kind == MC_CX ? cx_ctl_mask((ow >> 9) & 31, X0) : 0u;
      const int k = kind == MC_EXP ? (int)(ow >> 16) : 0;
      const double2 ph0 = kind == MC_EXP ? cs[2 * k] : make_double2(1, 0);
      const double2 ph1 = kind == MC_EXP ? cs[2 * k + 1] : make_double2(1, 0);
      if (m < 5) {  // lane bit: the partner is in this warp -- register shuffles, no barrier
        if (kind == MC_H) xlane_h(v, tid, m);
        else if (kind == MC_CX) xlane_cx(v, m, cm);
        else xlane_exp(v, tid, m, ph0, ph1);
      } else {  // warp bit: through shared memory
        if (kind == MC_H) xsmem_h(v, T, tid, m);
        else if (kind == MC_CX) xsmem_cx(v, T, tid, m, cm);
        else xsmem_exp(v, T, tid, m, ph0, ph1);
      }
    }
#pragma unroll
    for (int j = 0; j < kTileElems; j++) A[base | dep_lo_f | D.dep_hi_f[j]] = v[j];
  }
}

}  // namespace fs
