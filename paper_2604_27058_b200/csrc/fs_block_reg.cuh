// fs_block_reg.cuh -- warp-per-shot block engine with the active array in REGISTERS (k <= 10).
//
// The warp-per-shot block kernel (fs_block.cuh, G = 32) sweeps a shot's 2^k amplitudes through
// shared memory; at config 4's k = 9-10 segments it is 70 % of the program (profiles/
// r2_c4_launches.md) and its strided CX / CZ / H sweeps are shared-memory bound (bank conflicts,
// load latency).  Here element e of the array lives in register e >> 5 of lane e & 31 (NR = 2^(k_max
// - 5) registers of double2 per lane): an operation on an axis a >= 5 pairs registers inside a
// lane, an axis a < 5 pairs lanes through shuffles.  Register indices must be compile-time
// constants, so register-axis operations dispatch on the axis with a switch over unrolled cases.
//
// Results are bit-identical to fs_block.cuh: the same element-wise arithmetic, and the
// measurement reductions accumulate the same pairs in the same per-thread order (thread t sums
// pairs t, t + 32, ... -- gathered by shuffles when the axis is a lane bit) followed by the same
// shuffle tree.  The scalar VM (frames, records, noise, post-selection) is BlockCtx's, unchanged.
#pragma once
#include "fs_block.cuh"

namespace fs {

__device__ __forceinline__ double2 shfl_xor2(double2 x, int m) {
  return make_double2(__shfl_xor_sync(0xFFFFFFFFu, x.x, m), __shfl_xor_sync(0xFFFFFFFFu, x.y, m));
}
__device__ __forceinline__ double2 shfl_idx2(double2 x, int src) {
  return make_double2(__shfl_sync(0xFFFFFFFFu, x.x, src), __shfl_sync(0xFFFFFFFFu, x.y, src));
}

// dispatch a register-axis member template on R = axis - 5 (0..4)
#define FS_REG_DISPATCH(R, FN, ...)                     \
  switch (R) {                                          \
    case 0: this->template FN<0>(__VA_ARGS__); break;   \
    case 1: this->template FN<1>(__VA_ARGS__); break;   \
    case 2: this->template FN<2>(__VA_ARGS__); break;   \
    case 3: this->template FN<3>(__VA_ARGS__); break;   \
    default: this->template FN<4>(__VA_ARGS__); break;  \
  }

template <bool SPLITMIX, int NR>
struct BlockRegCtx : BlockCtx<SPLITMIX, 32> {
  using Base = BlockCtx<SPLITMIX, 32>;
  using Base::P;
  using Base::A;
  using Base::S;
  using Base::fx;
  using Base::fz;
  using Base::tid;
  using Base::si;
  using Base::gamma;
  using Base::sm;
  using Base::cpi;
  using Base::sh_alive;
  using Base::sh_k0;
  using Base::sh_k1;
  using Base::sh_branch;
  using Base::branch;
  using Base::renorm;
  double2 v[NR];

  __device__ __forceinline__ int lbit(int a) const { return (tid >> a) & 1; }  // lane part of element bit a < 5
  // bit a of element r * 32 + lane
  __device__ __forceinline__ int ebit(int r, int a) const { return a < 5 ? (int)((tid >> a) & 1) : (r >> (a - 5)) & 1; }
  __device__ __forceinline__ int nreg(uint32_t size) const { return size >= 32 ? (int)(size >> 5) : 1; }

  // register-axis bodies (RR = axis - 5, compile-time: every register index below is constant)
  template <int RR>
  __device__ __forceinline__ void h_reg(int nr) {
#pragma unroll
    for (int r = 0; r < NR; r++)
      if (!((r >> RR) & 1) && (r | (1 << RR)) < NR && (r | (1 << RR)) < nr) {
        const double2 lo = v[r], hi = v[r | (1 << RR)];
        v[r] = cscale(cadd(lo, hi), kInvSqrt2);
        v[r | (1 << RR)] = cscale(csub(lo, hi), kInvSqrt2);
      }
  }
  template <int RR>
  __device__ __forceinline__ void cx_reg(int nr, int a) {
#pragma unroll
    for (int r = 0; r < NR; r++)
      if (!((r >> RR) & 1) && (r | (1 << RR)) < NR && (r | (1 << RR)) < nr && ebit(r, a)) {
        const double2 t0 = v[r];
        v[r] = v[r | (1 << RR)];
        v[r | (1 << RR)] = t0;
      }
  }
  template <int RR>
  __device__ __forceinline__ void expand_reg(double2 ph0, double2 ph1) {
    constexpr int H = 1 << RR;  // live registers before the expand
#pragma unroll
    for (int r = 0; r < H; r++)
      if (r + H < NR) {
        const double2 x = v[r];
        v[r] = cmul(x, ph0);
        v[r + H] = cmul(x, ph1);
      }
  }
  template <int T, int RR>
  __device__ __forceinline__ void pair_reg(double2& a0, double2& a1) {
    constexpr uint32_t i0 = (((uint32_t)T & ~((1u << RR) - 1u)) << 1) | ((uint32_t)T & ((1u << RR) - 1u));
    a0 = v[i0 % NR];
    a1 = v[(i0 | (1u << RR)) % NR];
  }

  __device__ __forceinline__ void gate(int g, int va, int vb, int a, int b, uint32_t size) {
    const int nr = nreg(size);
    if (g == FS_G_S || g == FS_G_SDAG) {
      const double2 ph = make_double2(0.0, g == FS_G_S ? 1.0 : -1.0);
#pragma unroll
      for (int r = 0; r < NR; r++)
        if (r < nr && ebit(r, a)) v[r] = cmul(v[r], ph);
    } else if (g == FS_G_H) {
      if (a < 5) {
        const int m = 1 << a;
        const bool hi = (tid & m) != 0;
#pragma unroll
        for (int r = 0; r < NR; r++)
          if (r < nr) {
            const double2 p = shfl_xor2(v[r], m);
            v[r] = hi ? cscale(csub(p, v[r]), kInvSqrt2) : cscale(cadd(v[r], p), kInvSqrt2);
          }
      } else {
        FS_REG_DISPATCH(a - 5, h_reg, nr)
      }
    } else if (g == FS_G_CX) {  // control a, target b: elements with bit a set take their b-partner
      if (b < 5) {
        const int m = 1 << b;
#pragma unroll
        for (int r = 0; r < NR; r++)
          if (r < nr) {
            const double2 p = shfl_xor2(v[r], m);
            if (ebit(r, a)) v[r] = p;
          }
      } else {
        FS_REG_DISPATCH(b - 5, cx_reg, nr, a)
      }
    } else {  // CZ
#pragma unroll
      for (int r = 0; r < NR; r++)
        if (r < nr && ebit(r, a) && ebit(r, b)) v[r] = make_double2(-v[r].x, -v[r].y);
    }
    this->gate_frame(g, va, vb);
  }

  // Expand: element e < size -> e * ph0 and (e + size) * ph1
  __device__ __forceinline__ void expand(int virt, int fp, uint32_t size) {
    double2 ph0, ph1;
    this->parity_phases(virt, fp, 4, ph0, ph1);
    if (size < 32) {
      const int src = tid >= (int)size ? tid - (int)size : tid;
      const double2 x = shfl_idx2(v[0], src);
      v[0] = tid < (int)size ? cmul(v[0], ph0) : cmul(x, ph1);
    } else {
      FS_REG_DISPATCH(__ffs(size >> 5) - 1, expand_reg, ph0, ph1)
    }
    this->bar();
  }

  __device__ __forceinline__ void array_rot(int virt, int a, int fp, uint32_t size) {
    double2 e0, e1;
    this->parity_phases(virt, fp, 0, e0, e1);
    const int par = fx[virt] & 1;
    const double2 ph0 = par ? e1 : e0, ph1 = par ? e0 : e1;
    const int nr = nreg(size);
#pragma unroll
    for (int r = 0; r < NR; r++)
      if (r < nr) v[r] = cmul(v[r], ebit(r, a) ? ph1 : ph0);
    this->bar();
  }

  // the pair (element i0 = ins0(j, a), i0 + 2^a) of pair index j = tid + 32 t, as this lane sees it
  // in fs_block.cuh's loop (a0, a1); for a >= 5 it is in this lane's registers
  template <int T>
  __device__ __forceinline__ void pair_t(int a, double2& a0, double2& a1) {
    if (a < 5) {
      // i0 = ins0(tid + 32 t, a): lane ins0(tid, a) & 31, register 2 t + (tid >> 4)
      const int lane0 = (int)(ins0((uint32_t)tid, a) & 31u);
      const double2 x0 = shfl_idx2(v[(2 * T) % NR], lane0), x1 = shfl_idx2(v[(2 * T + 1) % NR], lane0);
      const double2 y0 = shfl_idx2(v[(2 * T) % NR], lane0 | (1 << a)), y1 = shfl_idx2(v[(2 * T + 1) % NR], lane0 | (1 << a));
      const bool up = (tid >> 4) & 1;
      a0 = up ? x1 : x0;
      a1 = up ? y1 : y0;
    } else {
      switch (a - 5) {
        case 0: pair_reg<T, 0>(a0, a1); break;
        case 1: pair_reg<T, 1>(a0, a1); break;
        case 2: pair_reg<T, 2>(a0, a1); break;
        case 3: pair_reg<T, 3>(a0, a1); break;
        default: pair_reg<T, 4>(a0, a1); break;
      }
    }
  }

  // MeasActive / MeasCollapse (fs_block.cuh measure(), same arithmetic and summation order)
  __device__ __forceinline__ bool measure(int i, bool collapse, int virt, int a, int rec, int flip, int ins4, int fp,
                                          uint32_t size) {
    const uint32_t half = size >> 1;
    double2 u00 = make_double2(1, 0), u01 = make_double2(0, 0), u10 = make_double2(0, 0), u11 = make_double2(1, 0);
    if (collapse) this->collapse_fparams(fp, u00, u01, u10, u11);
    double s1 = 0.0, sa = 0.0;
    auto acc = [&](double2 a0, double2 a1) {
      if (collapse) s1 = __dadd_rn(s1, cnorm2(cadd(cmul(a0, u10), cmul(u11, a1))));
      else s1 = __dadd_rn(s1, cnorm2(a1));
      sa = __dadd_rn(sa, __dadd_rn(cnorm2(a0), cnorm2(a1)));
    };
    // pairs j = tid + 32 t < half, t = 0 .. NR / 2 - 1 (NR >= 2), or one partial round
#pragma unroll
    for (int t = 0; t < (NR >= 2 ? NR / 2 : 1); t++) {
      double2 a0, a1;
      pair_tt(t, a, a0, a1);
      if ((uint32_t)(tid + 32 * t) < half) acc(a0, a1);
    }
    this->reduce2(s1, sa);
    this->meas_decide(i, collapse, virt, rec, flip, ins4, s1, sa, u00, u01, u10, u11);
    if (!sh_alive) return false;
    branch = sh_branch;
    if (collapse) {
      const double2 k0 = sh_k0, k1 = sh_k1;
      compact(a, half, [&](double2 a0, double2 a1) { return cadd(cmul(k0, a0), cmul(k1, a1)); });
    } else {
      const double s = sh_k0.x;
      const int dead = 1 - branch;
      const int nr = nreg(size);
#pragma unroll
      for (int r = 0; r < NR; r++)
        if (r < nr) {
          if (ebit(r, a) == dead) v[r] = make_double2(0.0, 0.0);
          else if (renorm) v[r] = cscale(v[r], s);
        }
    }
    this->bar();
    return true;
  }

  __device__ __forceinline__ void pair_tt(int t, int a, double2& a0, double2& a1) {
    // runtime t (unrolled loop index) -> compile-time template
    switch (t) {
#define FS_PT(T) case T: pair_t<T>(a, a0, a1); break;
      FS_PT(0) FS_PT(1) FS_PT(2) FS_PT(3) FS_PT(4) FS_PT(5) FS_PT(6) FS_PT(7)
      FS_PT(8) FS_PT(9) FS_PT(10) FS_PT(11) FS_PT(12) FS_PT(13) FS_PT(14) FS_PT(15)
#undef FS_PT
      default: break;
    }
  }

  // new element j < half = f(element ins0(j, a), element ins0(j, a) + 2^a); all pairs read
  // before any register is overwritten (new register r' reads registers >= r')
  // In place: new register t (pair j = tid + 32 t = new element j: lane tid, register t) reads
  // registers >= t only (2t, 2t + 1 for a lane axis; ins0(t, a - 5) and its partner for a
  // register axis), and every lane reads before it writes in the same instruction stream.
  template <class F>
  __device__ __forceinline__ void compact(int a, uint32_t half, F&& f) {
#pragma unroll
    for (int t = 0; t < (NR >= 2 ? NR / 2 : 1); t++) {
      double2 a0, a1;
      pair_tt(t, a, a0, a1);
      const double2 nv = f(a0, a1);
      if ((uint32_t)(tid + 32 * t) < half) v[t] = nv;
    }
  }

  __device__ __forceinline__ void retire(int virt, int a, uint32_t size) {
    const uint32_t half = size >> 1;
    const int br = sh_branch;
    compact(a, half, [&](double2 a0, double2 a1) { return br ? a1 : a0; });
    if (tid == 0) fx[virt] ^= (uint32_t)br;
    this->bar();
  }

  __device__ __forceinline__ void dump_cp(int j) {
    const size_t cs = (size_t)j * A.nshots + si;
    const int c = __ldg(A.cp_at + j);
    const uint32_t sz = 1u << (c > 0 ? __ldg(P.schedule + c - 1) : 0);
    double* dst = A.cp_amps + 2 * (__ldg(A.cp_off + j) + si * sz);
#pragma unroll
    for (int r = 0; r < NR; r++) {
      const uint32_t e = (uint32_t)r * 32 + tid;
      if (e < sz) { dst[2 * e] = v[r].x; dst[2 * e + 1] = v[r].y; }
    }
    for (int q = tid; q < P.n; q += 32) {
      A.cp_fx[cs * P.n + q] = (uint8_t)(fx[q] & 1u);
      A.cp_fz[cs * P.n + q] = (uint8_t)(fz[q] & 1u);
    }
    if (tid == 0) {
      A.cp_valid[cs] = 1;
      A.cp_gamma[2 * cs] = gamma.x;
      A.cp_gamma[2 * cs + 1] = gamma.y;
    }
  }
  __device__ __forceinline__ void dump_cps_at(int i) {
    bool any = false;
    while (cpi < A.ncp && __ldg(A.cp_at + cpi) == i) {
      dump_cp(cpi++);
      any = true;
    }
    if (any) this->bar();
  }

  __device__ __forceinline__ void dump_final(int upto) {
    const int kst = A.stop > 0 ? __ldg(P.schedule + A.stop - 1) : 0;
    const int kcur = upto > 0 ? __ldg(P.schedule + upto - 1) : 0;
    const uint32_t sz = 1u << kst, cur = 1u << kcur;
    if (A.t_amps) {
#pragma unroll
      for (int r = 0; r < NR; r++) {  // static register index per element (no dynamic v[])
        const uint32_t e = (uint32_t)r * 32 + tid;
        if (e < sz) {
          const double2 val = e < cur ? v[r] : make_double2(0.0, 0.0);
          A.t_amps[(si * sz + e) * 2] = val.x;
          A.t_amps[(si * sz + e) * 2 + 1] = val.y;
        }
      }
      for (uint32_t e = (uint32_t)NR * 32 + tid; e < sz; e += 32) {  // beyond this segment's capacity
        A.t_amps[(si * sz + e) * 2] = 0.0;
        A.t_amps[(si * sz + e) * 2 + 1] = 0.0;
      }
    }
    if (A.t_fx)
      for (int q = tid; q < P.n; q += 32) {
        A.t_fx[si * P.n + q] = (uint8_t)(fx[q] & 1u);
        A.t_fz[si * P.n + q] = (uint8_t)(fz[q] & 1u);
      }
    if (tid == 0) {
      if (A.t_gamma) { A.t_gamma[2 * si] = gamma.x; A.t_gamma[2 * si + 1] = gamma.y; }
      if (A.t_draws) A.t_draws[si] = SPLITMIX ? sm.count : 0u;
    }
  }

  __device__ __forceinline__ void interpret() {
    for (int i = S.seg_begin; i < S.seg_end; i++) {
      if (!sh_alive) break;
      if (A.ncp) dump_cps_at(i);
      int j = min(__ldg(P.next_array + i), S.seg_end);
      if (cpi < A.ncp) j = min(j, max(__ldg(A.cp_at + cpi), i));
      if (j > i) {
        this->scalar_run(i, j);
        i = j - 1;
        continue;
      }
      const int4 I0 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i);
      const int4 I1 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i + 1);
      const int ins[8] = {I0.x, I0.y, I0.z, I0.w, I1.x, I1.y, I1.z, I1.w};
      const int op = FS_OPCODE(I0.x);
      const int flip = FS_FLIP(I0.x);
      switch (op) {
        case FS_OP_FRAME: this->frame_matrix(__ldg(P.frame_mat_off + i)); break;
        case FS_OP_ARRAY_GATE: gate(ins[1], ins[2], ins[3], ins[4], ins[5], 1u << ins[6]); break;
        case FS_OP_EXPAND: expand(ins[1], ins[5], 1u << ins[6]); break;
        case FS_OP_ARRAY_ROT: array_rot(ins[1], ins[2], ins[5], 1u << ins[6]); break;
        case FS_OP_MEAS_ACTIVE:
        case FS_OP_MEAS_COLLAPSE:
          measure(i, op == FS_OP_MEAS_COLLAPSE, ins[1], ins[2], ins[3], flip, ins[4], ins[5], 1u << ins[6]);
          break;
        case FS_OP_RETIRE: retire(ins[1], ins[2], 1u << ins[6]); break;
        default: break;
      }
    }
    if (A.ncp && sh_alive) dump_cps_at(S.seg_end);
  }
};

#undef FS_REG_DISPATCH

// shot loop of a segment (block_run's structure with the array in registers): groups of one
// warp per shot, group_bytes of shared memory per group for the frame / slot / observable bytes
// shots (warps) per CTA: 8 when a lane holds 32 registers of amplitudes (register budget), else 16
template <int NR>
constexpr int block_reg_groups() { return NR >= 16 ? 8 : kBlockMaxGroups; }

template <bool SPLITMIX, int NR>
__global__ void __launch_bounds__(32 * block_reg_groups<NR>(), 1)
    block_reg_kernel(DevProg P, RunArgs A, SegArgs S, int karr, int group_bytes) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int group = threadIdx.x / 32, ngroups = blockDim.x / 32;
  uint32_t* fx = reinterpret_cast<uint32_t*>(smem_raw + (size_t)group * group_bytes);
  __shared__ double red1s[1], red2s[1];
  __shared__ double2 sh_k0s[kBlockMaxGroups], sh_k1s[kBlockMaxGroups];
  __shared__ int sh_alives[kBlockMaxGroups], sh_branchs[kBlockMaxGroups], sh_errs[kBlockMaxGroups];
  __shared__ uint32_t sh_slots[kBlockMaxGroups];
  const int tid = threadIdx.x % 32;
  (void)karr;
  for (uint32_t idx = blockIdx.x * ngroups + group; idx < S.n_in; idx += gridDim.x * ngroups) {
    const uint64_t si = S.first ? S.chunk0 + idx : S.in.shot[idx];
    if (si >= A.nshots) continue;  // uniform over the warp
    BlockRegCtx<SPLITMIX, NR> c{{P, A, S, nullptr, fx, fx + P.n, fx + 2 * P.n, fx + 2 * P.n + P.num_slots,
                                 sh_k0s[group], sh_k1s[group], sh_alives[group], sh_branchs[group], sh_errs[group],
                                 red1s, red2s, tid, idx, si, 0, 0, 0, !(A.flags & FS_NO_RENORM)}};
    c.shot = A.shot0 + si;
    c.wabs = c.shot >> 5;
    c.mylane = (int)(c.shot & 31);
    c.gamma = make_double2(1.0, 0.0);
    c.pend_site = -1;
    c.pend_lane = 0;
    c.pend_case = 0;
    c.branch = 0;
    c.coin_blk = -1;
    c.coin_b = make_uint4(0, 0, 0, 0);
    c.fmodes = A.fault_modes ? A.fault_modes + si * (size_t)P.E : nullptr;
    c.forced = A.forced ? A.forced + si * (size_t)P.R : nullptr;
    c.halt_i = -1;
    c.cpi = 0;
    if (A.ncp) {
      const int lo = S.seg_begin == 0 ? 0 : S.seg_begin + 1;
      while (c.cpi < A.ncp && __ldg(A.cp_at + c.cpi) < lo) c.cpi++;
    }
    if (tid == 0) {
      c.sh_alive = 1;
      c.sh_err = 0;
      if (SPLITMIX) c.sm.reset(A.seed, c.shot);
      else c.gen.init(A.seed, c.wabs);
    }
#pragma unroll
    for (int r = 0; r < NR; r++) c.v[r] = make_double2(0.0, 0.0);
    if (S.first) {
      for (int q = tid; q < 2 * P.n + P.num_slots + P.O; q += 32) fx[q] = 0;
      if (tid == 0) c.v[0] = make_double2(1.0, 0.0);
    } else {
      const StateStore& I = S.in;
      for (int b = tid; b < 2 * P.n; b += 32) fx[b] = (I.frame[(size_t)idx * S.nfw + (b >> 5)] >> (b & 31)) & 1u;
      for (int b = tid; b < P.num_slots; b += 32)
        c.slots[b] = (I.slotbits[(size_t)idx * S.nsw + (b >> 5)] >> (b & 31)) & 1u;
      for (int b = tid; b < P.O; b += 32) c.obsb[b] = (I.obsbits[(size_t)idx * S.now + (b >> 5)] >> (b & 31)) & 1u;
      const uint32_t sz = 1u << S.k_in;
#pragma unroll
      for (int r = 0; r < NR; r++) {
        const uint32_t e = (uint32_t)r * 32 + tid;
        if (e < sz) c.v[r] = I.amps[store_amp_index(idx, e, sz, I.shot_major)];
      }
      if (tid == 0) {
        c.gamma = I.gamma[idx];
        if (SPLITMIX) c.sm.count = I.smcount[idx];
        else {
          c.gen.step_no = I.gen_i[(size_t)idx * 6];
          c.gen.run = (int)I.gen_i[(size_t)idx * 6 + 1];
          c.gen.cl = (int)I.gen_i[(size_t)idx * 6 + 2];
          c.pend_site = (int)I.gen_i[(size_t)idx * 6 + 3];
          c.pend_lane = (int)I.gen_i[(size_t)idx * 6 + 4];
          c.pend_case = (int)I.gen_i[(size_t)idx * 6 + 5];
          c.gen.c = I.gen_c[idx];
        }
      }
    }
    c.bar();
    c.interpret();
    c.bar();
    const bool alive = c.sh_alive != 0;
    const bool errored = c.sh_err != 0;
    if ((S.last || !alive) && (A.t_fx || A.t_gamma || A.t_amps || A.t_draws)) {
      c.halt_i = __shfl_sync(0xFFFFFFFFu, c.halt_i, 0);
      c.dump_final(c.halt_i >= 0 ? c.halt_i : (S.last && alive ? A.stop : S.seg_end));
      c.bar();
    }
    if (tid == 0) {
      if (errored) {
        atomicOr(A.error + (si >> 5), 1u << (si & 31));
        atomicMax(A.status, c.sh_err);
      }
      if (S.last || !alive) {
        for (int o = 0; o < P.O; o++)
          if (c.obsb[o]) c.out_bit(A.obs + (size_t)o * A.W);
        if (alive && !errored) c.out_bit(A.accepted);
      }
    }
    if (!S.last && alive) {
      if (tid == 0) sh_slots[group] = atomicAdd(S.n_out, 1u);
      c.bar();
      const uint32_t slot = sh_slots[group];
      const StateStore& O = S.out;
      for (int j = tid; j < S.nfw; j += 32) {
        uint32_t vv = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < 2 * P.n; b++) vv |= (fx[b] & 1u) << (b & 31);
        O.frame[(size_t)slot * S.nfw + j] = vv;
      }
      for (int j = tid; j < S.nsw; j += 32) {
        uint32_t vv = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < P.num_slots; b++) vv |= (c.slots[b] & 1u) << (b & 31);
        O.slotbits[(size_t)slot * S.nsw + j] = vv;
      }
      for (int j = tid; j < S.now; j += 32) {
        uint32_t vv = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < P.O; b++) vv |= (c.obsb[b] & 1u) << (b & 31);
        O.obsbits[(size_t)slot * S.now + j] = vv;
      }
      const uint32_t sz = 1u << S.k_out;
#pragma unroll
      for (int r = 0; r < NR; r++) {
        const uint32_t e = (uint32_t)r * 32 + tid;
        if (e < sz) O.amps[store_amp_index(slot, e, sz, O.shot_major)] = c.v[r];
      }
      if (tid == 0) {
        O.shot[slot] = (uint32_t)si;
        O.gamma[slot] = c.gamma;
        if (SPLITMIX) O.smcount[slot] = c.sm.count;
        else {
          uint32_t* gi = O.gen_i + (size_t)slot * 6;
          gi[0] = c.gen.step_no; gi[1] = (uint32_t)c.gen.run; gi[2] = (uint32_t)c.gen.cl;
          gi[3] = (uint32_t)c.pend_site; gi[4] = (uint32_t)c.pend_lane; gi[5] = (uint32_t)c.pend_case;
          O.gen_c[slot] = c.gen.c;
        }
      }
    }
    c.bar();
  }
}

}  // namespace fs
