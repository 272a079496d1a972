// fs_block.cuh -- CTA-per-shot engine for segments whose active array is too large for a lane
// (2^k >= 512 amplitudes): the array of one shot lives in shared memory and every sweep is split
// across the group's threads; the scalar VM (frame bits, records, draws) runs on thread 0.
//
// Used by the segmented driver (post-selected programs, config 4): the survivor state store
// (fs_general.cuh StateStore) is engine-neutral, so consecutive segments may alternate between
// the lane-per-shot general engine (small k, many shots) and this engine (large k, few shots).
//
// Structure: BlockCtx holds one shot's state and implements every instruction; block_run is the
// shot loop (state load, survivor store, outputs) around an `exec(ctx)` functor.  block_kernel
// passes the instruction interpreter; the program-specialised segment kernels (fs_sampler.cu
// gen_block_source, NVRTC) pass straight-line code built from the same BlockCtx members.
#pragma once
#include "fs_general.cuh"

namespace fs {

// G threads per shot: G = 32 (warp per shot, several shots per CTA) or G = 256 (CTA per shot)
constexpr int kBlockMaxGroups = 16;  // warp-per-shot groups per CTA (bounded by shared memory)

template <bool SPLITMIX, int G>
struct BlockCtx {
  const DevProg& P;
  const RunArgs& A;
  const SegArgs& S;
  double2* amp;
  uint32_t *fx, *fz, *slots, *obsb;  // one shot: values 0/1 (fz = fx + n)
  double2& sh_k0;
  double2& sh_k1;
  int& sh_alive;
  int& sh_branch;
  int& sh_err;
  double* red1;
  double* red2;
  int tid;
  uint32_t idx;
  uint64_t si, shot, wabs;
  int mylane;
  bool renorm;
  // thread-0 scalar state
  double2 gamma;
  SplitMix sm;
  WordFaultGen gen;
  int pend_site, pend_lane, pend_case;
  int branch;
  int coin_blk;  // Philox coin block of ordinals 4b..4b+3, reused across coins
  uint4 coin_b;
  // trace mode (interpreter only): supplied draws, state dumps
  const int16_t* fmodes;  // [E] this shot's forced fault modes or NULL
  const int8_t* forced;   // [R] this shot's forced outcomes or NULL
  int cpi;                // next checkpoint
  int halt_i;             // instruction at which the shot halted (PostSelect), else -1

  __device__ __forceinline__ void put_rec(int rec, uint32_t bit) {
    const int col = __ldg(P.record_out + rec);
    if (col >= 0 && bit) out_bit(A.meas + (size_t)col * A.W);
    const int sl = __ldg(P.bit_slot + rec);
    if (sl >= 0) slots[sl] = bit;
    if (A.t_rec) A.t_rec[si * P.R + rec] = (uint8_t)bit;
  }
  __device__ __forceinline__ void fail(int code) {
    sh_err = code;
    sh_alive = 0;
  }

  __device__ __forceinline__ void bar() {
    if (G == 32) __syncwarp();
    else __syncthreads();
  }
  __device__ __forceinline__ void out_bit(uint32_t* row) { atomicOr(row + (si >> 5), 1u << (si & 31)); }

  // one scalar instruction of this shot (thread 0 only)
  __device__ __forceinline__ void scalar_step(int i) {
    const int4 I0 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i);
    const int4 I1 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i + 1);
    const int ins[8] = {I0.x, I0.y, I0.z, I0.w, I1.x, I1.y, I1.z, I1.w};
    const int op = FS_OPCODE(I0.x);
    const int flip = FS_FLIP(I0.x);
    switch (op) {
      case FS_OP_FRAME:
        for (int j = 0; j < ins[2]; j++) word_gate(fx, fz, __ldg(P.gates + ins[1] + j));
        break;
      case FS_OP_GAMMA_ROT: {
        const int par = fx[ins[1]] & 1;
        const double* f = P.fparams + ins[5] + 2 * par;
        gamma = cmul(gamma, make_double2(__ldg(f), __ldg(f + 1)));
        break;
      }
      case FS_OP_MEAS_DSTATIC:
      case FS_OP_MEAS_DRANDOM: {
        const int virt = ins[1], rec = ins[3];
        const int fo = forced ? (int)forced[rec] : -1;
        uint32_t bit;
        if (op == FS_OP_MEAS_DSTATIC) {
          bit = fx[virt] ^ (uint32_t)flip;
          if (fo >= 0 && (uint32_t)fo != bit) { fail(FS_ERR_SHOT_FORCED); break; }
        } else {
          const uint32_t pz = fz[virt];
          uint32_t coin;
          if (fo >= 0) {
            coin = (uint32_t)(fo ^ (int)pz ^ flip);
          } else if (SPLITMIX) {
            coin = (uint32_t)sm.bit();
          } else {
            if ((ins[2] >> 2) != coin_blk) {
              coin_blk = ins[2] >> 2;
              coin_b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), (uint32_t)coin_blk, TAG_COIN << 24, A.seed);
            }
            const int cj = ins[2] & 3;
            const uint32_t cw = cj == 0 ? coin_b.x : (cj == 1 ? coin_b.y : (cj == 2 ? coin_b.z : coin_b.w));
            coin = (cw >> mylane) & 1u;
          }
          bit = coin ^ pz ^ (uint32_t)flip;
          const uint32_t t = fx[virt];
          fx[virt] = fz[virt] ^ coin;
          fz[virt] = t;
          gamma = cscale(gamma, kInvSqrt2);
        }
        put_rec(rec, bit);
        break;
      }
      case FS_OP_COND_FRAME:
        if (slots[__ldg(P.bit_slot + ins[3])]) xor_paulis<false>(P, fx, fz, ins[1], ins[2], 1u);
        break;
      case FS_OP_NOISE:
        if (fmodes) {  // forced modes (runtime.py:587-601), draws as in the general engine
          ShotDraws d;
          d.splitmix = SPLITMIX;
          d.seed = A.seed;
          d.shot = shot;
          if (SPLITMIX) d.sm = sm;
          d.begin(i, TAG_FORCED);
          forced_faults_shot(P, fx, fz, 1u, ins, fmodes, d, 1, false);
          if (SPLITMIX) sm = d.sm;
        } else if (SPLITMIX) {
          hazard_shot(P, fx, fz, 1u, ins, sm, 1, false);
        } else {
          const int hi = ins[2];
          for (;;) {
            if (pend_site < 0) {
              int st_, ln_, cs_;
              const int r = gen.step(P, st_, ln_, cs_);
              if (r == 2) { pend_site = 0x7FFFFFFF; break; }
              if (r == 0) continue;
              pend_site = st_; pend_lane = ln_; pend_case = cs_;
            }
            if (pend_site >= hi) break;
            if (pend_lane == mylane) xor_case_strided(P, fx, fz, pend_case, 1u, 1, false);
            pend_site = -1;
          }
        }
        break;
      case FS_OP_DETECTOR:
      case FS_OP_OBSERVABLE: {
        uint32_t v = 0;
        for (int j = 0; j < ins[3]; j++) v ^= slots[__ldg(P.bit_slot + __ldg(P.reclists + ins[2] + j))];
        if (op == FS_OP_DETECTOR) {
          if (v) out_bit(A.det + (size_t)ins[1] * A.W);
          const int sl = __ldg(P.bit_slot + P.R + ins[1]);
          if (sl >= 0) slots[sl] = v;
        } else {
          obsb[ins[1]] ^= v;
        }
        break;
      }
      case FS_OP_POSTSELECT: {
        const int bid = ins[1] == 0 ? P.R + ins[2] : ins[2];
        if ((int)slots[__ldg(P.bit_slot + bid)] != ins[3]) {
          sh_alive = 0;
          halt_i = i;
        }
        break;
      }
      default: break;
    }
  }

  // scalar instructions [i, j) on thread 0, one barrier at the end
  __device__ __forceinline__ void scalar_run(int i, int j) {
    if (tid == 0)
      for (int t = i; t < j && sh_alive; t++) scalar_step(t);
    bar();
  }

  // FrameGates i as its GF(2) matrix (warp-wide ballots + popcounts)
  __device__ __forceinline__ void frame_matrix(int mo) {
    if (tid < 32) {
      const int n2 = 2 * P.n;
      uint32_t v[4], o[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int bb = tid + 32 * k;
        v[k] = __ballot_sync(0xFFFFFFFFu, bb < n2 && (fx[bb] & 1u));
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int r = tid + 32 * k;
        o[k] = 0u;
        if (r < n2) {
          const uint4 row = __ldg(reinterpret_cast<const uint4*>(P.frame_mat + mo) + r);
          o[k] = (uint32_t)(__popc(row.x & v[0]) + __popc(row.y & v[1]) + __popc(row.z & v[2]) +
                            __popc(row.w & v[3])) & 1u;
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (tid + 32 * k < n2) fx[tid + 32 * k] = o[k];
    }
    bar();
  }

  // frame side of an ArrayGate (thread 0), then the barrier that ends the instruction
  __device__ __forceinline__ void gate_frame(int g, int va, int vb) {
    if (tid == 0) {
      uint32_t t;
      switch (g) {
        case FS_G_S: case FS_G_SDAG: fz[va] ^= fx[va]; break;
        case FS_G_H: t = fx[va]; fx[va] = fz[va]; fz[va] = t; break;
        case FS_G_CX: fx[vb] ^= fx[va]; fz[va] ^= fz[vb]; break;
        case FS_G_CZ: fz[vb] ^= fx[va]; fz[va] ^= fx[vb]; break;
      }
    }
    bar();
  }

  __device__ __forceinline__ void gate(int g, int va, int vb, int a, int b, uint32_t size) {
    if (g == FS_G_S || g == FS_G_SDAG) {
      const double2 ph = make_double2(0.0, g == FS_G_S ? 1.0 : -1.0);
      for (uint32_t j = tid; j < size / 2; j += G) {
        const uint32_t id = ins0(j, a) | (1u << a);
        amp[id] = cmul(amp[id], ph);
      }
    } else if (g == FS_G_H) {
      const uint32_t st = 1u << a;
      for (uint32_t j = tid; j < size / 2; j += G) {
        const uint32_t i0 = ins0(j, a);
        const double2 lo = amp[i0], hi = amp[i0 + st];
        amp[i0] = cscale(cadd(lo, hi), kInvSqrt2);
        amp[i0 + st] = cscale(csub(lo, hi), kInvSqrt2);
      }
    } else {
      const int lo_ax = a < b ? a : b, hi_ax = a < b ? b : a;
      for (uint32_t j = tid; j < size / 4; j += G) {
        const uint32_t id = ins0(ins0(j, lo_ax), hi_ax) | (1u << a);
        const uint32_t jd = id | (1u << b);
        if (g == FS_G_CX) {
          const double2 t0 = amp[id];
          amp[id] = amp[jd];
          amp[jd] = t0;
        } else {
          const double2 v = amp[jd];
          amp[jd] = make_double2(-v.x, -v.y);
        }
      }
    }
    gate_frame(g, va, vb);
  }

  // Expand / ArrayRot phases selected by the frame parity of `virt`
  __device__ __forceinline__ void parity_phases(int virt, int fp, int stride, double2& ph0, double2& ph1) {
    const int par = fx[virt] & 1;
    const double* f = P.fparams + fp + stride * par;
    ph0 = make_double2(__ldg(f), __ldg(f + 1));
    ph1 = make_double2(__ldg(f + 2), __ldg(f + 3));
  }

  __device__ __forceinline__ void expand(int virt, int fp, uint32_t size) {
    double2 ph0, ph1;
    parity_phases(virt, fp, 4, ph0, ph1);
    for (uint32_t j = tid; j < size; j += G) {
      const double2 v = amp[j];
      amp[j] = cmul(v, ph0);
      amp[size + j] = cmul(v, ph1);
    }
    bar();
  }

  __device__ __forceinline__ void array_rot(int virt, int a, int fp, uint32_t size) {
    double2 e0, e1;
    parity_phases(virt, fp, 0, e0, e1);
    const int par = fx[virt] & 1;
    const double2 ph0 = par ? e1 : e0, ph1 = par ? e0 : e1;
    for (uint32_t j = tid; j < size; j += G) amp[j] = cmul(amp[j], ((j >> a) & 1) ? ph1 : ph0);
    bar();
  }

  // x with its sign bit flipped where m has bit 31 set
  static __device__ __forceinline__ double flipsign(double x, uint32_t m) {
    return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
  }

  // A star group (fs_sampler.cu fs_program_create): the ArrayGates CX(a, .), CZ(a, .), S / S_DAG(a),
  // [H(a)], [ArrayRot] of a localisation run in one sweep.  Elements with bit a clear stay; element
  // j with bit a set becomes i^(pw + 2 parity(j & Mz)) * old[j ^ M]; then H on a, then the
  // ArrayRot phases.  The group's frame matrix has been applied (ArrayRot reads the parity after it).
  // SWAP = pw odd (the factor is +-i: real and imaginary parts trade places).
  template <bool SWAP>
  __device__ __forceinline__ void star_group_t(int a, uint32_t M, uint32_t Mz, uint32_t pw, bool hasH, bool hasAR,
                                               int ar_virt, int ar_axis, int ar_fp, uint32_t size) {
    const uint32_t A_ = 1u << a;
    double2 ph0 = make_double2(1.0, 0.0), ph1 = ph0;
    if (hasAR) {
      double2 e0, e1;
      parity_phases(ar_virt, ar_fp, 0, e0, e1);
      const int par = fx[ar_virt] & 1;
      ph0 = par ? e1 : e0;
      ph1 = par ? e0 : e1;
    }
    // v * i^(pw + 2 par): the x sign flips iff par ^ (pw in {1, 2}), the y sign iff par ^ (pw >= 2)
    const uint32_t cx = (pw == 1u || pw == 2u) ? 0x80000000u : 0u, cy = pw >= 2u ? 0x80000000u : 0u;
    auto hiphase = [&](uint32_t id, double2 v) {
      const uint32_t sg = (uint32_t)__popc(id & Mz) << 31;
      return make_double2(flipsign(SWAP ? v.y : v.x, sg ^ cx), flipsign(SWAP ? v.x : v.y, sg ^ cy));
    };
    auto finish = [&](uint32_t i0, double2 lo, double2 hi) {  // lo at i0, hi at i0 | A_
      if (hasH) {
        const double2 s = cscale(cadd(lo, hi), kInvSqrt2), d = cscale(csub(lo, hi), kInvSqrt2);
        lo = s;
        hi = d;
      }
      if (hasAR) {
        lo = cmul(lo, ((i0 >> ar_axis) & 1u) ? ph1 : ph0);
        hi = cmul(hi, (((i0 | A_) >> ar_axis) & 1u) ? ph1 : ph0);
      }
      amp[i0] = lo;
      amp[i0 | A_] = hi;
    };
    const bool touch_lo = hasH || hasAR;
    if (M == 0u) {
      for (uint32_t j = tid; j < size / 2; j += G) {
        const uint32_t i0 = ins0(j, a);
        const double2 hi = hiphase(i0 | A_, amp[i0 | A_]);
        if (touch_lo) finish(i0, amp[i0], hi);
        else amp[i0 | A_] = hi;
      }
    } else {
      const int m = __ffs((int)M) - 1;
      const int lo_ax = a < m ? a : m, hi_ax = a < m ? m : a;
      for (uint32_t j = tid; j < size / 4; j += G) {
        const uint32_t i0 = ins0(ins0(j, lo_ax), hi_ax), i1 = i0 ^ M;  // bit a clear in both
        const double2 h0 = amp[i1 | A_], h1 = amp[i0 | A_];
        const double2 n0 = hiphase(i0 | A_, h0), n1 = hiphase(i1 | A_, h1);
        if (touch_lo) {
          finish(i0, amp[i0], n0);
          finish(i1, amp[i1], n1);
        } else {
          amp[i0 | A_] = n0;
          amp[i1 | A_] = n1;
        }
      }
    }
    bar();
  }
  __device__ __forceinline__ void star_group(int a, uint32_t M, uint32_t Mz, uint32_t pw, bool hasH, bool hasAR,
                                             int ar_virt, int ar_axis, int ar_fp, uint32_t size) {
    if (pw & 1u) star_group_t<true>(a, M, Mz, pw, hasH, hasAR, ar_virt, ar_axis, ar_fp, size);
    else star_group_t<false>(a, M, Mz, pw, hasH, hasAR, ar_virt, ar_axis, ar_fp, size);
  }

  // group gi of the descriptor table: its frame matrix, then the sweep
  __device__ __forceinline__ int run_group(int gi) {
    const int4 D0 = __ldg(reinterpret_cast<const int4*>(P.fuse) + 2 * gi);
    const int4 D1 = __ldg(reinterpret_cast<const int4*>(P.fuse) + 2 * gi + 1);
    frame_matrix(D1.w);
    star_group(D0.y & 0xFF, (uint32_t)D0.z, (uint32_t)D0.w, (uint32_t)D1.x & 3u, (D1.x & 4) != 0, (D1.x & 8) != 0,
               D1.y & 0xFFFF, D1.y >> 16, D1.z, 1u << (D0.y >> 8));
    return D0.x;
  }

  // fixed-order tree: element t += element t + w for w = G/2 .. 1 (same pairs either way)
  __device__ __forceinline__ void reduce2(double& s1, double& sa) {
    if (G == 32) {
#pragma unroll
      for (int w = 16; w; w >>= 1) {
        const double o1 = __shfl_down_sync(0xFFFFFFFFu, s1, w), o2 = __shfl_down_sync(0xFFFFFFFFu, sa, w);
        if (tid < w) {
          s1 = __dadd_rn(s1, o1);
          sa = __dadd_rn(sa, o2);
        }
      }
    } else {
      red1[tid] = s1;
      red2[tid] = sa;
      bar();
      for (int w = G >> 1; w; w >>= 1) {
        if (tid < w) {
          red1[tid] = __dadd_rn(red1[tid], red1[tid + w]);
          red2[tid] = __dadd_rn(red2[tid], red2[tid + w]);
        }
        bar();
      }
      s1 = red1[0];
      sa = red2[0];
    }
  }

  // measurement of instruction i from the reduced (p1, p_all) (thread 0): branch, record,
  // Kraus factors for the compaction; ends with the barrier that publishes them
  __device__ __forceinline__ void meas_decide(int i, bool collapse, int virt, int rec, int flip, int ins4,
                                              double s1, double sa, double2 u00, double2 u01, double2 u10,
                                              double2 u11) {
    if (tid == 0) {
      if (collapse) {
        const int po = ins4 >> 8, pc = ins4 & 0xFF;
        for (int j = 0; j < pc; j++) word_gate(fx, fz, __ldg(P.gates + po + j));
      }
      double p1 = s1, p_all = sa;
      const int parity = fx[virt] & 1;
      int bad = 0;
      if (p1 != p1) bad = FS_ERR_SHOT_NAN;
      if (collapse || !renorm) p1 = p_all > 0 ? __ddiv_rn(p1, p_all) : 0.0;
      if (p1 < 0.0) p1 = 0.0;
      else if (p1 > 1.0) p1 = 1.0;
      const int fo = forced ? (int)forced[rec] : -1;
      int br;
      double pb;
      if (fo < 0) {
        double u;
        if (SPLITMIX) u = sm.uniform();
        else {
          const uint4 o = philox((uint32_t)shot, (uint32_t)(shot >> 32), (uint32_t)i, TAG_BORN << 24, A.seed);
          u = u64_to_unit(((uint64_t)o.y << 32) | o.x);
        }
        br = u < p1 ? 1 : 0;
        pb = br ? p1 : __dsub_rn(1.0, p1);
        if (pb < kBranchFloor) { br ^= 1; pb = __dsub_rn(1.0, pb); }
      } else {  // forced outcome (runtime.py:383-386, :476-479)
        br = fo ^ parity ^ flip;
        pb = br ? p1 : __dsub_rn(1.0, p1);
        if (!bad && pb < kBranchFloor) bad = FS_ERR_SHOT_FORCED;
      }
      if (bad) {
        sh_err = bad;
        sh_alive = 0;
      } else {
        const uint32_t recbit = (uint32_t)(br ^ parity ^ flip);
        put_rec(rec, recbit);
        if (collapse) {
          const double scale = renorm ? __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(pb, p_all))) : 1.0;
          sh_k0 = br == 0 ? cscale(u00, scale) : cscale(u10, scale);
          sh_k1 = br == 0 ? cscale(u01, scale) : cscale(u11, scale);
          fx[virt] ^= (uint32_t)br;
        } else {
          sh_k0 = make_double2(renorm ? __ddiv_rn(1.0, __dsqrt_rn(pb)) : 1.0, 0.0);
        }
        sh_branch = br;
        if (renorm) gamma = cscale(gamma, __dsqrt_rn(pb));
      }
    }
    bar();
  }

  __device__ __forceinline__ void collapse_fparams(int fp, double2& u00, double2& u01, double2& u10, double2& u11) {
    const double* f = P.fparams + fp;
    u00 = make_double2(__ldg(f), __ldg(f + 1));
    u01 = make_double2(__ldg(f + 2), __ldg(f + 3));
    u10 = make_double2(__ldg(f + 4), __ldg(f + 5));
    u11 = make_double2(__ldg(f + 6), __ldg(f + 7));
  }

  // MeasActive / MeasCollapse; returns false when the shot stopped (error)
  __device__ __forceinline__ bool measure(int i, bool collapse, int virt, int a, int rec, int flip, int ins4, int fp,
                                          uint32_t size) {
    const uint32_t half = size >> 1, st = 1u << a;
    double2 u00 = make_double2(1, 0), u01 = make_double2(0, 0), u10 = make_double2(0, 0), u11 = make_double2(1, 0);
    if (collapse) collapse_fparams(fp, u00, u01, u10, u11);
    // (p1, p_all) partial sums in a fixed order per thread, then a fixed-order tree
    double s1 = 0.0, sa = 0.0;
    for (uint32_t j = tid; j < half; j += G) {
      const uint32_t i0 = ins0(j, a);
      const double2 a0 = amp[i0], a1 = amp[i0 + st];
      if (collapse) s1 = __dadd_rn(s1, cnorm2(cadd(cmul(a0, u10), cmul(u11, a1))));
      else s1 = __dadd_rn(s1, cnorm2(a1));
      sa = __dadd_rn(sa, __dadd_rn(cnorm2(a0), cnorm2(a1)));
    }
    reduce2(s1, sa);
    meas_decide(i, collapse, virt, rec, flip, ins4, s1, sa, u00, u01, u10, u11);
    if (!sh_alive) return false;
    branch = sh_branch;
    if (collapse) {  // in place, one strip of G outputs at a time: strip b reads indices >= its
                     // own outputs, all above what earlier strips wrote
      const double2 k0 = sh_k0, k1 = sh_k1;
      for (uint32_t b0 = 0; b0 < half; b0 += G) {
        const uint32_t j = b0 + tid;
        double2 val = make_double2(0.0, 0.0);
        if (j < half) {
          const uint32_t i0 = ins0(j, a);
          val = cadd(cmul(k0, amp[i0]), cmul(k1, amp[i0 + st]));
        }
        bar();
        if (j < half) amp[j] = val;
        bar();
      }
    } else {
      const double s = sh_k0.x;
      const uint32_t dead = 1u - (uint32_t)branch;
      for (uint32_t j = tid; j < size; j += G) {
        if (((j >> a) & 1) == dead) amp[j] = make_double2(0.0, 0.0);
        else if (renorm) amp[j] = cscale(amp[j], s);
      }
    }
    bar();
    return true;
  }

  __device__ __forceinline__ void retire(int virt, int a, uint32_t size) {
    const uint32_t half = size >> 1;
    const int br = sh_branch;
    for (uint32_t b0 = 0; b0 < half; b0 += G) {  // in place, strip by strip (as collapse)
      const uint32_t j = b0 + tid;
      double2 val = make_double2(0.0, 0.0);
      if (j < half) val = amp[ins0(j, a) + ((uint32_t)br << a)];
      bar();
      if (j < half) amp[j] = val;
      bar();
    }
    if (tid == 0) fx[virt] ^= (uint32_t)br;
    bar();
  }

  // trace: state after instructions [0, cp_at[j]) (all threads: amplitudes; thread 0: scalars)
  __device__ __forceinline__ void dump_cp(int j) {
    const size_t cs = (size_t)j * A.nshots + si;
    const int c = __ldg(A.cp_at + j);
    const uint32_t sz = 1u << (c > 0 ? __ldg(P.schedule + c - 1) : 0);
    double* dst = A.cp_amps + 2 * (__ldg(A.cp_off + j) + si * sz);
    for (uint32_t e = tid; e < sz; e += G) {
      dst[2 * e] = amp[e].x;
      dst[2 * e + 1] = amp[e].y;
    }
    for (int q = tid; q < P.n; q += G) {
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
    if (any) bar();
  }

  // the interpreter: instructions [seg_begin, seg_end) of the segment
  __device__ __forceinline__ void interpret() {
    for (int i = S.seg_begin; i < S.seg_end; i++) {
      if (!sh_alive) break;
      if (A.ncp) dump_cps_at(i);
      int j = min(__ldg(P.next_array + i), S.seg_end);
      if (cpi < A.ncp) j = min(j, max(__ldg(A.cp_at + cpi), i));  // scalar runs stop at checkpoints
      if (j > i) {  // a run of scalar instructions
        scalar_run(i, j);
        i = j - 1;
        continue;
      }
      const int4 I0 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i);
      const int4 I1 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i + 1);
      const int ins[8] = {I0.x, I0.y, I0.z, I0.w, I1.x, I1.y, I1.z, I1.w};
      const int op = FS_OPCODE(I0.x);
      const int flip = FS_FLIP(I0.x);
      switch (op) {
        case FS_OP_FRAME: frame_matrix(__ldg(P.frame_mat_off + i)); break;  // next_array stops here only with a matrix
        case FS_OP_ARRAY_GATE: {
          const int gi = S.fuse ? __ldg(P.fuse_at + i) : -1;
          if (gi >= 0) i += run_group(gi) - 1;
          else gate(ins[1], ins[2], ins[3], ins[4], ins[5], 1u << ins[6]);
          break;
        }
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

  // trace: final state of a shot that ended (halted, raised or finished) in this segment
  __device__ __forceinline__ void dump_final(int upto) {
    const int kst = A.stop > 0 ? __ldg(P.schedule + A.stop - 1) : 0;
    const int kcur = upto > 0 ? __ldg(P.schedule + upto - 1) : 0;
    const uint32_t sz = 1u << kst, cur = 1u << kcur;
    if (A.t_amps)
      for (uint32_t e = tid; e < sz; e += G) {
        const double2 v = e < cur ? amp[e] : make_double2(0.0, 0.0);
        A.t_amps[(si * sz + e) * 2] = v.x;
        A.t_amps[(si * sz + e) * 2 + 1] = v.y;
      }
    if (A.t_fx)
      for (int q = tid; q < P.n; q += G) {
        A.t_fx[si * P.n + q] = (uint8_t)(fx[q] & 1u);
        A.t_fz[si * P.n + q] = (uint8_t)(fz[q] & 1u);
      }
    if (tid == 0) {
      if (A.t_gamma) { A.t_gamma[2 * si] = gamma.x; A.t_gamma[2 * si + 1] = gamma.y; }
      if (A.t_draws) A.t_draws[si] = SPLITMIX ? sm.count : 0u;
    }
  }
};

// the shot loop of a segment: state load, exec(ctx) for the instructions, outputs and survivor
// store.  Launch: G * ngroups threads, group_bytes of dynamic shared memory per group.
template <bool SPLITMIX, int G, class Exec>
__device__ __forceinline__ void block_run(const DevProg& P, const RunArgs& A, const SegArgs& S, int karr,
                                          int group_bytes, Exec&& exec) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t cap = 1u << karr;
  const int group = threadIdx.x / G, ngroups = blockDim.x / G;
  double2* amp = reinterpret_cast<double2*>(smem_raw + (size_t)group * group_bytes);
  uint32_t* fx = reinterpret_cast<uint32_t*>(amp + cap);
  // reduction scratch only for the CTA-per-shot form (warp groups reduce with shuffles)
  __shared__ double red1s[G == 256 ? 256 : 1], red2s[G == 256 ? 256 : 1];
  __shared__ double2 sh_k0s[kBlockMaxGroups], sh_k1s[kBlockMaxGroups];
  __shared__ int sh_alives[kBlockMaxGroups], sh_branchs[kBlockMaxGroups], sh_errs[kBlockMaxGroups];
  __shared__ uint32_t sh_slots[kBlockMaxGroups];
  const int tid = threadIdx.x % G;
  for (uint32_t idx = blockIdx.x * ngroups + group; idx < S.n_in; idx += gridDim.x * ngroups) {
    const uint64_t si = S.first ? S.chunk0 + idx : S.in.shot[idx];
    if (si >= A.nshots) continue;  // uniform over the block
    BlockCtx<SPLITMIX, G> c{P, A, S, amp, fx, fx + P.n, fx + 2 * P.n, fx + 2 * P.n + P.num_slots,
                            sh_k0s[group], sh_k1s[group], sh_alives[group], sh_branchs[group], sh_errs[group],
                            red1s, red2s, tid, idx, si, 0, 0, 0, !(A.flags & FS_NO_RENORM)};
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
    if (S.first) {
      for (int q = tid; q < 2 * P.n + P.num_slots + P.O; q += G) fx[q] = 0;
      if (tid == 0) amp[0] = make_double2(1.0, 0.0);
    } else {
      const StateStore& I = S.in;
      // the array goes global -> shared asynchronously (16 B per request, no register staging)
      // while the frame bits and the scalar state load
      const uint32_t sz = 1u << S.k_in, icap = 1u << S.k_in;
      for (uint32_t j = tid; j < sz; j += G) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(amp + j);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(I.amps + store_amp_index(idx, j, icap, I.shot_major)) : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      for (int b = tid; b < 2 * P.n; b += G) fx[b] = (I.frame[(size_t)idx * S.nfw + (b >> 5)] >> (b & 31)) & 1u;
      for (int b = tid; b < P.num_slots; b += G)
        c.slots[b] = (I.slotbits[(size_t)idx * S.nsw + (b >> 5)] >> (b & 31)) & 1u;
      for (int b = tid; b < P.O; b += G) c.obsb[b] = (I.obsbits[(size_t)idx * S.now + (b >> 5)] >> (b & 31)) & 1u;
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
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    c.bar();
    exec(c);
    c.bar();
    const bool alive = c.sh_alive != 0;
    const bool errored = c.sh_err != 0;
    if ((S.last || !alive) && (A.t_fx || A.t_gamma || A.t_amps || A.t_draws)) {
      c.halt_i = __shfl_sync(0xFFFFFFFFu, c.halt_i, 0);  // thread 0's (G >= 32: lane 0 of warp 0)
      if (G == 256) {
        __shared__ int sh_halt;
        if (tid == 0) sh_halt = c.halt_i;
        c.bar();
        c.halt_i = sh_halt;
      }
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
    if (!S.last && alive) {  // survivor: compact into the output store
      if (tid == 0) sh_slots[group] = atomicAdd(S.n_out, 1u);
      c.bar();
      const uint32_t slot = sh_slots[group];
      const StateStore& O = S.out;
      for (int j = tid; j < S.nfw; j += G) {
        uint32_t v = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < 2 * P.n; b++) v |= (fx[b] & 1u) << (b & 31);
        O.frame[(size_t)slot * S.nfw + j] = v;
      }
      for (int j = tid; j < S.nsw; j += G) {
        uint32_t v = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < P.num_slots; b++) v |= (c.slots[b] & 1u) << (b & 31);
        O.slotbits[(size_t)slot * S.nsw + j] = v;
      }
      for (int j = tid; j < S.now; j += G) {
        uint32_t v = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < P.O; b++) v |= (c.obsb[b] & 1u) << (b & 31);
        O.obsbits[(size_t)slot * S.now + j] = v;
      }
      const uint32_t sz = 1u << S.k_out;
      for (uint32_t j = tid; j < sz; j += G) O.amps[store_amp_index(slot, j, sz, O.shot_major)] = amp[j];
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

template <bool SPLITMIX, int G>
// warp groups: shared memory admits one CTA per SM at the k >= 9 this form runs (13-16 groups),
// so the register budget is 128 per thread
__global__ void __launch_bounds__(G == 32 ? 32 * kBlockMaxGroups : 256, G == 32 ? 1 : 4)
    block_kernel(DevProg P, RunArgs A, SegArgs S, int karr, int group_bytes) {
  block_run<SPLITMIX, G>(P, A, S, karr, group_bytes, [](BlockCtx<SPLITMIX, G>& c) { c.interpret(); });
}

}  // namespace fs
