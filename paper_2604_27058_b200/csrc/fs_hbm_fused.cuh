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
  int8_t T[kTileBits];   // physical axis of each tile bit
  int8_t base[32];       // live physical axes outside the tile (tile index bits)
  uint32_t dep_hi[kTileElems];  // physical offset of element j = tid + 256 * j, high part
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

// pass op staged in shared memory: kind | xa << 4 | xb << 9 | diag_run << 16, where xa / xb are
// positions in the extended local index X = tid | j << 8 | tile << 12 (tile bits 0..11, then the
// tile index bits = the pass's base axes); ca / cb = the op's constants with the shot's parity
// already applied (ROT: factor for bit 0 / 1; EXPAND: phase of the bit-0 / bit-1 half)
struct StagedOp {
  uint32_t w, pad;
  double2 ca, cb;
};
constexpr int kPassMaxOps = kTileThreads;

__device__ __forceinline__ uint32_t reg_mask(int R) {  // j in [0,16) with bit R set
  return (uint32_t)((0xFF00F0F0CCCCAAAAull >> (16 * R)) & 0xFFFFu);
}

// 16-bit mask over j of the elements whose bit at extended position x is set
__device__ __forceinline__ uint32_t pos_mask(int x, uint32_t X0) {
  return (unsigned)(x - 8) < 4u ? reg_mask(x - 8) : (((X0 >> x) & 1u) ? 0xFFFFu : 0u);
}

__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

// a run of diagonal ops (CZ, S, S_DAG, ROT) on the thread's 16 elements.  Diagonal ops commute,
// so the run is accumulated as  v[j] *= i^P(j) * g * prod_{R : bit R of j} d_R  with the power P
// held as two 16-bit planes over j (bit 0 in Lm, bit 1 in Hm) and applied once at the end.
__device__ __forceinline__ void diag_run_apply(double2 (&v)[kTileElems], const StagedOp* __restrict__ so, int run,
                                               uint32_t X0) {
  uint32_t Lm = 0, Hm = 0, rreg = 0;
  bool grot = false;
  double2 g = make_double2(1, 0);
  double2 d[4];
#pragma unroll
  for (int q = 0; q < 4; q++) d[q] = make_double2(1, 0);
  for (int r = 0; r < run; r++) {
    const uint32_t w = so[r].w;
    const int kind = w & 15, xa = (w >> 4) & 31, xb = (w >> 9) & 31;
    const uint32_t ma = pos_mask(xa, X0);
    if (kind == TO_CZ) {
      Hm ^= ma & pos_mask(xb, X0);
    } else if (kind == TO_S) {  // P += 1 where bit set
      const uint32_t c = Lm & ma;
      Lm ^= ma;
      Hm ^= c;
    } else if (kind == TO_SDAG) {  // P -= 1 where bit set
      const uint32_t b = ~Lm & ma;
      Lm ^= ma;
      Hm ^= b;
    } else {  // ROT
      const double2 ca = so[r].ca, cb = so[r].cb;
      if ((unsigned)(xa - 8) < 4u) {
        const int R = xa - 8;
        g = cmul(g, ca);
        const double2 rat = cdiv(cb, ca);
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (q == R) d[q] = cmul(d[q], rat);
        rreg |= 1u << R;
      } else {
        g = cmul(g, ma ? cb : ca);
        grot = true;
      }
    }
  }
  Lm &= 0xFFFFu;
  Hm &= 0xFFFFu;
  if (Lm | Hm) {
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
  if (rreg) {
    double2 t01[4], t23[4];
    t01[0] = g;
    t01[1] = cmul(g, d[0]);
    t01[2] = cmul(g, d[1]);
    t01[3] = cmul(t01[1], d[1]);
    t23[1] = d[2];
    t23[2] = d[3];
    t23[3] = cmul(d[2], d[3]);
#pragma unroll
    for (int j = 0; j < kTileElems; j++) {
      const double2 f = (j >> 2) ? cmul(t01[j & 3], t23[j >> 2]) : t01[j & 3];
      v[j] = cmul(v[j], f);
    }
  } else if (grot) {
#pragma unroll
    for (int j = 0; j < kTileElems; j++) v[j] = cmul(v[j], g);
  }
}

__global__ void __launch_bounds__(kTileThreads, 2) hbm_fused_pass_kernel(HbmState H, const PassDesc D,
                                                                        const TileOp* __restrict__ ops, uint32_t W) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* T = reinterpret_cast<double2*>(smem_raw);
  StagedOp* so = reinterpret_cast<StagedOp*>(smem_raw + sizeof(double2) * (1 << kTileBits));
  const uint32_t shot = blockIdx.y;
  const uint32_t w = shot >> 5, bit = 1u << (shot & 31);
  if (!(H.alive[w] & bit)) return;
  const uint32_t tid = threadIdx.x;
  const int nops = D.nops;
  if ((int)tid < nops) {  // stage this pass's ops, resolving the shot's parities
    const TileOp& o = ops[D.op_off + tid];
    StagedOp s;
    s.w = (uint32_t)o.kind | (uint32_t)(o.la & 31) << 4 | (uint32_t)(o.lb & 31) << 9 | (uint32_t)o.diag_run << 16;
    s.pad = 0;
    s.ca = o.c0;
    s.cb = o.c1;
    if (o.kind == TO_ROT || o.kind == TO_EXPAND) {
      const bool par = (H.par[(size_t)o.instr * W + w] & bit) != 0;
      if (o.kind == TO_ROT && par) { s.ca = o.c1; s.cb = o.c0; }
      if (o.kind == TO_EXPAND && par) { s.ca = o.c2; s.cb = o.c3; }
    }
    so[tid] = s;
  }
  uint32_t dep_lo = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) dep_lo |= ((tid >> i) & 1u) << D.T[i];
  const uint64_t ntiles = 1ull << D.nbase;
  double2* __restrict__ A = H.amps + (size_t)shot * H.cap;
  __syncthreads();
  double2 v[kTileElems];
  for (uint64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const uint64_t base = deposit_bits(ti, D.base, D.nbase);
    const uint32_t X0 = tid | (uint32_t)(ti << kTileBits);
#pragma unroll
    for (int j = 0; j < kTileElems; j++) v[j] = A[base | dep_lo | D.dep_hi[j]];
    for (int k = 0; k < nops; k++) {
      const uint32_t ow = so[k].w;
      const int kind = ow & 15;
      const int run = (ow >> 16) & 255;
      if (run > 0) {
        diag_run_apply(v, so + k, run, X0);
        k += run - 1;
        continue;
      }
      const int xa = (ow >> 4) & 31, xb = (ow >> 9) & 31;
      const int m = kind == TO_CX ? xb : xa;  // mixing bit (always inside the tile)
      if (m >= 8) {  // register bit: no data exchange
        const int R = m - 8;
        if (kind == TO_H) {
          if (R == 0) reg_h<0>(v); else if (R == 1) reg_h<1>(v); else if (R == 2) reg_h<2>(v); else reg_h<3>(v);
        } else if (kind == TO_CX) {
          const bool creg = (unsigned)(xa - 8) < 4u;
          const int c = creg ? xa - 8 : (int)((X0 >> xa) & 1u);
          const int ck = creg ? 0 : 3;
          if (!creg && !c) continue;
          if (R == 0) reg_cx<0>(v, ck, c, tid, 0); else if (R == 1) reg_cx<1>(v, ck, c, tid, 0);
          else if (R == 2) reg_cx<2>(v, ck, c, tid, 0); else reg_cx<3>(v, ck, c, tid, 0);
        } else {
          const double2 ph0 = so[k].ca, ph1 = so[k].cb;
          if (R == 0) reg_expand<0>(v, ph0, ph1); else if (R == 1) reg_expand<1>(v, ph0, ph1);
          else if (R == 2) reg_expand<2>(v, ph0, ph1); else reg_expand<3>(v, ph0, ph1);
        }
        continue;
      }
      // thread bit: exchange with partner thread tid ^ (1 << m) through shared memory
#pragma unroll
      for (int j = 0; j < kTileElems; j++) T[tid + kTileThreads * j] = v[j];
      __syncthreads();
      const uint32_t ptid = tid ^ (1u << m);
      const int mine_bit = (tid >> m) & 1;
      if (kind == TO_H) {
#pragma unroll
        for (int j = 0; j < kTileElems; j++) {
          const double2 pv = T[ptid + kTileThreads * j];
          v[j] = mine_bit ? cscale(csub(pv, v[j]), kInvSqrt2) : cscale(cadd(v[j], pv), kInvSqrt2);
        }
      } else if (kind == TO_CX) {
        const uint32_t cm = pos_mask(xa, X0);
#pragma unroll
        for (int j = 0; j < kTileElems; j++)
          if ((cm >> j) & 1u) v[j] = T[ptid + kTileThreads * j];
      } else {  // expand: bit-1 half gets the bit-0 partner times ph1
        const double2 ph0 = so[k].ca, ph1 = so[k].cb;
#pragma unroll
        for (int j = 0; j < kTileElems; j++) {
          const double2 pv = T[ptid + kTileThreads * j];
          v[j] = mine_bit ? cmul(pv, ph1) : cmul(v[j], ph0);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < kTileElems; j++) A[base | dep_lo | D.dep_hi[j]] = v[j];
  }
}

}  // namespace fs
