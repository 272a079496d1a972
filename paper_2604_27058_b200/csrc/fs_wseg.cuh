// fs_wseg.cuh -- warp- and CTA-per-shot segments of the block engine, fully specialised (NVRTC).
//
// The interpreter form (fs_block.cuh block_kernel<.., 32>) keeps one shot's frame as one shared
// word per bit and runs every scalar instruction (FrameGates, dormant measurements, CondFrame,
// noise, detectors) on thread 0 between warp barriers -- at the k = 9-10 segments of config 4 that
// scalar VM, not the array sweeps, is most of the time (profiles/r2_c4_block_ncu.md).  Here the
// whole segment is straight-line code generated per program (fs_sampler.cu gen_segment_w):
//
//   * the frame of the shot is bit-packed in four registers (2n <= 128 bits: x_q at bit q, z_q at
//     bit n + q -- the survivor store's own layout) that every lane holds: scalar instructions are
//     executed redundantly by all 32 lanes, so there is no shared-memory frame, no barrier and no
//     instruction decode; a CondFrame or a noise case is four XORs with a mask (immediates, or
//     one 16-byte load from the host-built per-case table), a frame gate two or three register
//     instructions at constant bit positions;
//   * record / detector slots and observables are one register each;
//   * array sweeps are the block engine's (same per-thread order of partial sums, same tree);
//   * the measurement decision is taken by every lane from the broadcast sums.
//
// Philox stream, no trace inputs or outputs (those run the interpreter).  State in and out through
// the engine-neutral survivor store (fs_general.cuh StateStore).
#pragma once
#include "fs_block.cuh"

// complex multiply of the specialised segment kernels: the fused form (as in fs_jit_general:
// records unchanged, amplitudes within the last ulp of the interpreters') unless the including
// source asks for the interpreters' own
#ifndef FS_SEG_CMUL
#define FS_SEG_CMUL cmul_f
#endif

namespace fs {

// Scalar state of one shot and the scalar instructions on it (shared by the warp-per-shot segments
// below, where all 32 lanes hold the same shot and `writer` is lane 0, and the lane-per-shot
// segments of fs_lseg.cuh, where every lane is its own shot's writer)
struct SCtx {
  const DevProg& P;
  const RunArgs& A;
  const SegArgs& S;
  uint64_t si, shot, wabs;
  int mylane;
  bool renorm, writer;
  uint32_t F[4];        // packed frame
  uint32_t slots, obs;  // packed record / detector slots, observables
  int alive, err;
  WordFaultGen gen;
  int pend_site, pend_lane, pend_case, pend_certain;
  double pend_x;
  int coin_blk;
  uint4 coin_b;
  int branch;

  __device__ __forceinline__ SCtx(const DevProg& P_, const RunArgs& A_, const SegArgs& S_, uint64_t si_, bool writer_)
      : P(P_), A(A_), S(S_), si(si_), shot(A_.shot0 + si_), renorm(!(A_.flags & FS_NO_RENORM)), writer(writer_) {
    wabs = shot >> 5;
    mylane = (int)(shot & 31);
    alive = 1;
    err = 0;
    pend_site = -1;
    pend_lane = 0;
    pend_case = 0;
    pend_certain = 0;
    pend_x = 0.0;
    branch = 0;
    coin_blk = -1;
    coin_b = make_uint4(0, 0, 0, 0);
    gen.init(A.seed, wabs);
#pragma unroll
    for (int k = 0; k < 4; k++) F[k] = 0u;
    slots = 0u;
    obs = 0u;
  }

  __device__ __forceinline__ uint32_t fbit(int b) const { return (F[b >> 5] >> (b & 31)) & 1u; }
  __device__ __forceinline__ void fxor(int b, uint32_t v) { F[b >> 5] ^= v << (b & 31); }
  // frame bit dst ^= frame bit src: the source word shifted by the difference of the two bit
  // positions, masked to the destination bit (a shift and one three-input logic instruction when
  // the positions are constants, as in the generated code)
  __device__ __forceinline__ void xor_from(int dst, int src) {
    const int d = (src & 31) - (dst & 31);
    const uint32_t w = F[src >> 5];
    F[dst >> 5] ^= (d >= 0 ? w >> d : w << -d) & (1u << (dst & 31));
  }
  // frame gates on bit positions (x_a, z_a, x_b, z_b are positions in the packed frame)
  __device__ __forceinline__ void g_s(int xa, int za) { xor_from(za, xa); }
  __device__ __forceinline__ void g_h(int xa, int za) {  // x <-> z
    xor_from(xa, za);
    xor_from(za, xa);
    xor_from(xa, za);
  }
  __device__ __forceinline__ void g_cx(int xa, int za, int xb, int zb) {
    xor_from(xb, xa);
    xor_from(za, zb);
  }
  __device__ __forceinline__ void g_cz(int xa, int za, int xb, int zb) {
    xor_from(zb, xa);
    xor_from(za, xb);
  }
  __device__ __forceinline__ void g_swap(int xa, int za, int xb, int zb) {
    xor_from(xa, xb);
    xor_from(xb, xa);
    xor_from(xa, xb);
    xor_from(za, zb);
    xor_from(zb, za);
    xor_from(za, zb);
  }
  __device__ __forceinline__ void xor_mask(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
    F[0] ^= m0; F[1] ^= m1; F[2] ^= m2; F[3] ^= m3;
  }

  __device__ __forceinline__ void out_bit(uint32_t* row) {
    if (writer) atomicOr(row + (si >> 5), 1u << (si & 31));
  }
  // record bit: user column col (or -1), slot sl (or -1)
  __device__ __forceinline__ void put_rec(int col, int sl, uint32_t bit) {
    if (col >= 0 && bit) out_bit(A.meas + (size_t)col * A.W);
    if (sl >= 0) slots = (slots & ~(1u << sl)) | (bit << sl);
  }

  __device__ __forceinline__ void meas_dstatic(int xq, int flip, int col, int sl) { put_rec(col, sl, fbit(xq) ^ (uint32_t)flip); }
  __device__ __forceinline__ void meas_drandom(int xq, int zq, int ord, int flip, int col, int sl) {
    if ((ord >> 2) != coin_blk) {
      coin_blk = ord >> 2;
      coin_b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), (uint32_t)coin_blk, TAG_COIN << 24, A.seed);
    }
    const int cj = ord & 3;
    const uint32_t cw = cj == 0 ? coin_b.x : (cj == 1 ? coin_b.y : (cj == 2 ? coin_b.z : coin_b.w));
    const uint32_t coin = (cw >> mylane) & 1u, px = fbit(xq), pz = fbit(zq);
    fxor(xq, px ^ pz ^ coin);  // x <- z ^ coin
    fxor(zq, pz ^ px);         // z <- old x
    put_rec(col, sl, coin ^ pz ^ (uint32_t)flip);
  }
  __device__ __forceinline__ void detector(uint32_t v, int d, int sl) {
    if (v) out_bit(A.det + (size_t)d * A.W);
    if (sl >= 0) slots = (slots & ~(1u << sl)) | (v << sl);
  }

  // NoiseBlock over sites < hi: the word's fault stream, this shot's lane.  The same stream and the
  // same faults as fs_block.cuh scalar_step, but a candidate is resolved (thinning test, case pick:
  // dependent table loads) only if it is this shot's; another lane's candidate is just a place to
  // stop at (pend_case == -2: unresolved)
  __device__ __forceinline__ void noise(int hi) {
    for (;;) {
      if (pend_site < 0) {
        int st_, ln_, ce_;
        double x_;
        const int r = gen.step_cand(P, st_, ln_, x_, ce_);
        if (r == 2) { pend_site = 0x7FFFFFFF; break; }
        if (r == 0) continue;
        pend_site = st_; pend_lane = ln_; pend_case = -2; pend_x = x_; pend_certain = ce_;
      }
      if (pend_site >= hi) break;
      if (pend_lane == mylane) {
        const int cs = pend_case == -2 ? WordFaultGen::resolve(P, pend_site, pend_x, pend_certain) : pend_case;
        if (cs >= 0) {
          const uint4 m = __ldg(P.case_mask + cs);
          xor_mask(m.x, m.y, m.z, m.w);
        }
      }
      pend_site = -1;
    }
  }
  // before the state goes to the survivor store: other engines expect a resolved pending fault; a
  // candidate of another lane or one that thinning drops is no fault of this shot, the next
  // NoiseBlock just goes on stepping
  __device__ __forceinline__ void settle_pending() {
    if (pend_site >= 0 && pend_site != 0x7FFFFFFF && pend_case == -2) {
      const int cs = pend_lane == mylane ? WordFaultGen::resolve(P, pend_site, pend_x, pend_certain) : -1;
      if (cs >= 0) pend_case = cs;
      else { pend_site = -1; pend_case = 0; }
    }
  }

  // survivor state in / out of the engine-neutral store (everything but the amplitudes)
  __device__ __forceinline__ void load_scalars(const StateStore& I, uint32_t idx) {
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (k < S.nfw) F[k] = I.frame[(size_t)idx * S.nfw + k];
    if (S.nsw) slots = I.slotbits[(size_t)idx * S.nsw];
    if (S.now) obs = I.obsbits[(size_t)idx * S.now];
    gen.step_no = I.gen_i[(size_t)idx * 6];
    gen.run = (int)I.gen_i[(size_t)idx * 6 + 1];
    gen.cl = (int)I.gen_i[(size_t)idx * 6 + 2];
    pend_site = (int)I.gen_i[(size_t)idx * 6 + 3];
    pend_lane = (int)I.gen_i[(size_t)idx * 6 + 4];
    pend_case = (int)I.gen_i[(size_t)idx * 6 + 5];
    gen.c = I.gen_c[idx];
  }
};

// G threads per shot: 32 (one warp, warp barriers and shuffles), 64 .. 256 (warps of one CTA behind a
// named barrier; per-warp partial sums and broadcast words go through the shot's scratch `scr`)
template <int G>
struct WCtxT : SCtx {
  double2* amp;
  double* scr;  // G > 32: 2 * (G / 32) doubles of partial sums, then 4 words
  int tid, bar_id;

  __device__ __forceinline__ WCtxT(const DevProg& P_, const RunArgs& A_, const SegArgs& S_, double2* amp_, double* scr_, int tid_,
                                   int bar_id_, uint64_t si_)
      : SCtx(P_, A_, S_, si_, tid_ == 0), amp(amp_), scr(scr_), tid(tid_), bar_id(bar_id_) {}

  // NoiseBlock (SCtx::noise) with the draws of 32 consecutive steps of the word's stream made at
  // once: lane j of each warp holds the two draws of step cb0 + j (one Philox block and one ln per
  // lane instead of per step), the walk over the steps reads them by shuffles.  All lanes of a
  // warp hold the same shot, so they walk in lockstep; the stream position that goes to the
  // survivor store is the plain one (step_no, run, cl, c), the batch is dropped at the segment end.
  uint32_t cb0 = 0u;
  bool chave = false;
  double cL = 0.0, cU = 0.0;
  __device__ __forceinline__ void noise(int hi) {
    const int ln = tid & 31;
    for (;;) {
      if (pend_site < 0) {
        if (gen.run >= P.num_runs) { pend_site = 0x7FFFFFFF; break; }
        if (!chave || gen.step_no - cb0 >= 32u) {
          cb0 = gen.step_no;
          const uint4 b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), 0u, (TAG_NOISE << 24) | (cb0 + (uint32_t)ln), A.seed);
          cU = u64_to_unit(((uint64_t)b.w << 32) | b.z);
          cL = ln_unit(((uint64_t)b.y << 32) | b.x);
          chave = true;
        }
        const int src = (int)(gen.step_no - cb0);
        const double L = __shfl_sync(0xFFFFFFFFu, cL, src), u2 = __shfl_sync(0xFFFFFFFFu, cU, src);
        int st_, ln_, ce_;
        double x_;
        const int r = gen.step_with(P, L, u2, st_, ln_, x_, ce_);
        if (r == 0) continue;
        pend_site = st_; pend_lane = ln_; pend_case = -2; pend_x = x_; pend_certain = ce_;
      }
      if (pend_site >= hi) break;
      if (pend_lane == mylane) {
        const int cs = pend_case == -2 ? WordFaultGen::resolve(P, pend_site, pend_x, pend_certain) : pend_case;
        if (cs >= 0) {
          const uint4 m = __ldg(P.case_mask + cs);
          xor_mask(m.x, m.y, m.z, m.w);
        }
      }
      pend_site = -1;
    }
  }

  // barrier of the shot's threads
  __device__ __forceinline__ void sync() const {
    if (G == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(G) : "memory");
  }

  // sweeps ------------------------------------------------------------------------------------
  __device__ __forceinline__ void gate(int g, int a, int b, uint32_t size) {
    if (g == FS_G_S || g == FS_G_SDAG) {
      const double2 ph = make_double2(0.0, g == FS_G_S ? 1.0 : -1.0);
      for (uint32_t j = tid; j < size / 2; j += G) {
        const uint32_t id = ins0(j, a) | (1u << a);
        amp[id] = FS_SEG_CMUL(amp[id], ph);
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
    sync();
  }

  __device__ __forceinline__ void expand(uint32_t size, double2 ph0, double2 ph1) {
    for (uint32_t j = tid; j < size; j += G) {
      const double2 v = amp[j];
      amp[j] = FS_SEG_CMUL(v, ph0);
      amp[size + j] = FS_SEG_CMUL(v, ph1);
    }
    sync();
  }

  __device__ __forceinline__ void array_rot(int a, uint32_t size, double2 ph0, double2 ph1) {
    for (uint32_t j = tid; j < size; j += G) amp[j] = FS_SEG_CMUL(amp[j], ((j >> a) & 1) ? ph1 : ph0);
    sync();
  }

  // star group (fs_block.cuh star_group_t); ph0 / ph1 = the closing ArrayRot's phases for bit 0 / 1
  template <bool SWAP>
  __device__ __forceinline__ void star(int a, uint32_t M, uint32_t Mz, uint32_t pw, bool hasH, bool hasAR, int ar_axis,
                                       double2 ph0, double2 ph1, uint32_t size) {
    const uint32_t A_ = 1u << a;
    const uint32_t cx = (pw == 1u || pw == 2u) ? 0x80000000u : 0u, cy = pw >= 2u ? 0x80000000u : 0u;
    auto hiphase = [&](uint32_t id, double2 v) {
      const uint32_t sg = (uint32_t)__popc(id & Mz) << 31;
      return make_double2(BlockCtx<false, 32>::flipsign(SWAP ? v.y : v.x, sg ^ cx),
                          BlockCtx<false, 32>::flipsign(SWAP ? v.x : v.y, sg ^ cy));
    };
    auto finish = [&](uint32_t i0, double2 lo, double2 hi) {
      if (hasH) {
        const double2 s = cscale(cadd(lo, hi), kInvSqrt2), d = cscale(csub(lo, hi), kInvSqrt2);
        lo = s;
        hi = d;
      }
      if (hasAR) {
        lo = FS_SEG_CMUL(lo, ((i0 >> ar_axis) & 1u) ? ph1 : ph0);
        hi = FS_SEG_CMUL(hi, (((i0 | A_) >> ar_axis) & 1u) ? ph1 : ph0);
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
        const uint32_t i0 = ins0(ins0(j, lo_ax), hi_ax), i1 = i0 ^ M;
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
    sync();
  }

  // MeasActive / MeasCollapse (fs_block.cuh measure + meas_decide); xv = frame bit of the measured
  // virtual qubit's X part (the collapse pre-gates have been applied by the caller).  Returns false
  // when the shot stopped (NaN).
  template <bool COLLAPSE>
  __device__ __forceinline__ bool measure(int i, int xv, int a, int flip, int col, int sl, uint32_t size, double2 u00,
                                          double2 u01, double2 u10, double2 u11) {
    const uint32_t half = size >> 1, st = 1u << a;
    double s1 = 0.0, sa = 0.0;
    for (uint32_t j = tid; j < half; j += G) {
      const uint32_t i0 = ins0(j, a);
      const double2 a0 = amp[i0], a1 = amp[i0 + st];
      if (COLLAPSE) s1 = __dadd_rn(s1, cnorm2(cadd(FS_SEG_CMUL(a0, u10), FS_SEG_CMUL(u11, a1))));
      else s1 = __dadd_rn(s1, cnorm2(a1));
      sa = __dadd_rn(sa, __dadd_rn(cnorm2(a0), cnorm2(a1)));
    }
#pragma unroll
    for (int w = 16; w; w >>= 1) {  // the block engine's tree: element t += element t + w
      const double o1 = __shfl_down_sync(0xFFFFFFFFu, s1, w), o2 = __shfl_down_sync(0xFFFFFFFFu, sa, w);
      if ((tid & 31) < w) {
        s1 = __dadd_rn(s1, o1);
        sa = __dadd_rn(sa, o2);
      }
    }
    double p1, p_all;
    if (G == 32) {
      p1 = __shfl_sync(0xFFFFFFFFu, s1, 0);
      p_all = __shfl_sync(0xFFFFFFFFu, sa, 0);
    } else {  // warp sums in warp order, by every thread
      if ((tid & 31) == 0) {
        scr[2 * (tid >> 5)] = s1;
        scr[2 * (tid >> 5) + 1] = sa;
      }
      sync();
      p1 = scr[0];
      p_all = scr[1];
#pragma unroll
      for (int w = 1; w < G / 32; w++) {
        p1 = __dadd_rn(p1, scr[2 * w]);
        p_all = __dadd_rn(p_all, scr[2 * w + 1]);
      }
      sync();
    }
    const uint32_t parity = fbit(xv);
    if (p1 != p1) {
      err = FS_ERR_SHOT_NAN;
      alive = 0;
      return false;
    }
    if (COLLAPSE || !renorm) p1 = p_all > 0 ? __ddiv_rn(p1, p_all) : 0.0;
    if (p1 < 0.0) p1 = 0.0;
    else if (p1 > 1.0) p1 = 1.0;
    const uint4 o = philox((uint32_t)shot, (uint32_t)(shot >> 32), (uint32_t)i, TAG_BORN << 24, A.seed);
    const double u = u64_to_unit(((uint64_t)o.y << 32) | o.x);
    int br = u < p1 ? 1 : 0;
    double pb = br ? p1 : __dsub_rn(1.0, p1);
    if (pb < kBranchFloor) { br ^= 1; pb = __dsub_rn(1.0, pb); }
    put_rec(col, sl, (uint32_t)br ^ parity ^ (uint32_t)flip);
    branch = br;
    if (COLLAPSE) {
      const double scale = renorm ? __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(pb, p_all))) : 1.0;
      const double2 k0 = br == 0 ? cscale(u00, scale) : cscale(u10, scale);
      const double2 k1 = br == 0 ? cscale(u01, scale) : cscale(u11, scale);
      fxor(xv, (uint32_t)br);
      for (uint32_t b0 = 0; b0 < half; b0 += G) {  // in place, strip by strip
        const uint32_t j = b0 + tid;
        double2 val = make_double2(0.0, 0.0);
        if (j < half) {
          const uint32_t i0 = ins0(j, a);
          val = cadd(FS_SEG_CMUL(k0, amp[i0]), FS_SEG_CMUL(k1, amp[i0 + st]));
        }
        sync();
        if (j < half) amp[j] = val;
        sync();
      }
    } else {
      const double s = renorm ? __ddiv_rn(1.0, __dsqrt_rn(pb)) : 1.0;
      const uint32_t dead = 1u - (uint32_t)br;
      for (uint32_t j = tid; j < size; j += G) {
        if (((j >> a) & 1) == dead) amp[j] = make_double2(0.0, 0.0);
        else if (renorm) amp[j] = cscale(amp[j], s);
      }
      sync();
    }
    return true;
  }

  __device__ __forceinline__ void retire(int xv, int a, uint32_t size) {
    const uint32_t half = size >> 1;
    for (uint32_t b0 = 0; b0 < half; b0 += G) {
      const uint32_t j = b0 + tid;
      double2 val = make_double2(0.0, 0.0);
      if (j < half) val = amp[ins0(j, a) + ((uint32_t)branch << a)];
      sync();
      if (j < half) amp[j] = val;
      sync();
    }
    fxor(xv, (uint32_t)branch);
  }
};

// the shot loop of a specialised warp-per-shot segment (fs_block.cuh block_run without the shared
// frame): one warp per shot, `group_bytes` of dynamic shared memory per warp for the array
template <int G, int KARR, class Exec>
__device__ __forceinline__ void wseg_run(const DevProg& P, const RunArgs& A, const SegArgs& S, int group_bytes,
                                         Exec&& exec) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int group = threadIdx.x / G, ngroups = blockDim.x / G, tid = threadIdx.x % G;
  double2* amp = reinterpret_cast<double2*>(smem_raw + (size_t)group * group_bytes);
  // the shot's scratch follows its array (fs_sampler.cu launch_block_kernel leaves >= 256 bytes)
  double* scr = reinterpret_cast<double*>(smem_raw + (size_t)group * group_bytes + ((size_t)16 << KARR));
  uint32_t* scrw = reinterpret_cast<uint32_t*>(scr + 2 * (G / 32));
  const int bar_id = ngroups == 1 ? 0 : group + 1;
  for (uint32_t idx = blockIdx.x * ngroups + group; idx < S.n_in; idx += gridDim.x * ngroups) {
    const uint64_t si = S.first ? S.chunk0 + idx : S.in.shot[idx];
    if (si >= A.nshots) continue;
    WCtxT<G> c(P, A, S, amp, scr, tid, bar_id, si);
    double2 gamma = make_double2(1.0, 0.0);
    if (S.first) {
      if (tid == 0) amp[0] = make_double2(1.0, 0.0);
    } else {
      const StateStore& I = S.in;
      const uint32_t sz = 1u << S.k_in;
      const double2* const src = I.amps + store_amp_index(idx, 0, sz, I.shot_major);
      const uint32_t sstride = I.shot_major ? 1u : 32u;
      for (uint32_t j = tid; j < sz; j += G) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(amp + j);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + (size_t)j * sstride) : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      c.load_scalars(I, idx);
      gamma = I.gamma[idx];
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    c.sync();
    exec(c);
    c.sync();
    const bool alive = c.alive != 0, errored = c.err != 0;
    if (tid == 0 && errored) {
      atomicOr(A.error + (si >> 5), 1u << (si & 31));
      atomicMax(A.status, c.err);
    }
    if (S.last || !alive) {
      for (int o = 0; o < P.O; o++)
        if ((c.obs >> o) & 1u) c.out_bit(A.obs + (size_t)o * A.W);
      if (alive && !errored) c.out_bit(A.accepted);
    }
    if (!S.last && alive) {  // survivor: compact into the output store
      c.settle_pending();
      uint32_t slot = 0;
      if (tid == 0) slot = atomicAdd(S.n_out, 1u);
      if (G == 32) slot = __shfl_sync(0xFFFFFFFFu, slot, 0);
      else {
        if (tid == 0) scrw[0] = slot;
        c.sync();
        slot = scrw[0];
      }
      const StateStore& O = S.out;
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (k < S.nfw && tid == k) O.frame[(size_t)slot * S.nfw + k] = c.F[k];
      const uint32_t sz = 1u << S.k_out;
      // element j of the slot: base + j * stride (shot-major or lane-interleaved store)
      double2* const dst = O.amps + store_amp_index(slot, 0, sz, O.shot_major);
      const uint32_t dstride = O.shot_major ? 1u : 32u;
      for (uint32_t j = tid; j < sz; j += G) dst[(size_t)j * dstride] = amp[j];
      if (tid == 0) {
        if (S.nsw) O.slotbits[(size_t)slot * S.nsw] = c.slots;
        if (S.now) O.obsbits[(size_t)slot * S.now] = c.obs;
        O.shot[slot] = (uint32_t)si;
        O.gamma[slot] = gamma;
        uint32_t* gi = O.gen_i + (size_t)slot * 6;
        gi[0] = c.gen.step_no; gi[1] = (uint32_t)c.gen.run; gi[2] = (uint32_t)c.gen.cl;
        gi[3] = (uint32_t)c.pend_site; gi[4] = (uint32_t)c.pend_lane; gi[5] = (uint32_t)c.pend_case;
        O.gen_c[slot] = c.gen.c;
      }
    }
    c.sync();
  }
}

}  // namespace fs
