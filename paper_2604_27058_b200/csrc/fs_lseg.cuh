// fs_lseg.cuh -- lane-per-shot segments of the segmented engine, fully specialised (NVRTC).
//
// Segments whose active array stays small (k < the block engine's threshold) are scalar work:
// FrameGates, dormant measurements, CondFrame, noise, detectors, a few Expands (config 4's first
// three segments hold no ArrayGate at all).  The interpreter form (fs_general.cuh general_kernel
// <.., SEG>) keeps the 32 shots of a warp bit-sliced in shared memory and runs FrameGates and the
// survivor packing on lane 0 / bit by bit.  Here every lane owns one shot outright:
//
//   * the frame is the shot's packed words (SCtx, fs_wseg.cuh -- the survivor store's own layout):
//     a frame gate is two or three register instructions at compile-time bit positions, a noise
//     case or CondFrame four XORs, restore and save are plain word loads / stores;
//   * the active array is a per-thread array indexed by constants where the generated code unrolls
//     (k <= kLsegUnrollK: registers), else thread-local memory (lane-interleaved by the hardware,
//     L1 / L2 resident);
//   * no warp collective inside a segment body: lanes may leave early (NaN, post-selection) and
//     meet again at the survivor compaction.
//
// Same instruction semantics and the same draws as every other engine (Philox stream; sums run
// sequentially per shot as in the interpreter's lane-per-shot form).  No trace inputs or outputs
// (those run the interpreter).
#pragma once
#include "fs_wseg.cuh"

namespace fs {

constexpr int kLsegUnrollK = 4;  // arrays up to 2^4 amplitudes are unrolled into registers

template <int KARR, int NLAZY>
struct LCtx : SCtx {
  double2* __restrict__ arr;  // the shot's array: a thread-local array of 2^KARR in lseg_run
  // Expands after the segment's last array-reading instruction are not executed: their phase pairs
  // (picked at their program point) wait here and are applied when the survivor is saved
  double2 lz0[NLAZY > 0 ? NLAZY : 1], lz1[NLAZY > 0 ? NLAZY : 1];

  __device__ __forceinline__ LCtx(const DevProg& P_, const RunArgs& A_, const SegArgs& S_, uint64_t si_, double2* arr_)
      : SCtx(P_, A_, S_, si_, true), arr(arr_) {}

  // ArrayGate G on axes AX (and BX), array of 2^K
  template <int G, int AX, int BX, int K>
  __device__ __forceinline__ void gate() {
    constexpr uint32_t size = 1u << K;
    if (G == FS_G_S || G == FS_G_SDAG) {
#pragma unroll(K <= kLsegUnrollK ? (1 << K) : 4)
      for (uint32_t j = 0; j < size / 2; j++) {
        const uint32_t id = ins0(j, AX) | (1u << AX);
        const double2 v = arr[id];
        arr[id] = G == FS_G_S ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
      }
    } else if (G == FS_G_H) {
      constexpr uint32_t st = 1u << AX;
#pragma unroll(K <= kLsegUnrollK ? (1 << K) : 4)
      for (uint32_t j = 0; j < size / 2; j++) {
        const uint32_t i0 = ins0(j, AX);
        const double2 lo = arr[i0], hi = arr[i0 + st];
        arr[i0] = cscale(cadd(lo, hi), kInvSqrt2);
        arr[i0 + st] = cscale(csub(lo, hi), kInvSqrt2);
      }
    } else {
      constexpr int lo_ax = AX < BX ? AX : BX, hi_ax = AX < BX ? BX : AX;
#pragma unroll(K <= kLsegUnrollK ? (1 << K) : 4)
      for (uint32_t j = 0; j < size / 4; j++) {
        const uint32_t id = ins0(ins0(j, lo_ax), hi_ax) | (1u << AX);
        const uint32_t jd = id | (1u << BX);
        if (G == FS_G_CX) {
          const double2 t0 = arr[id];
          arr[id] = arr[jd];
          arr[jd] = t0;
        } else {
          const double2 v = arr[jd];
          arr[jd] = make_double2(-v.x, -v.y);
        }
      }
    }
  }

  // Expand of an array of 2^K (k_before): amplitudes j and 2^K + j from amplitude j
  template <int K>
  __device__ __forceinline__ void expand(double2 ph0, double2 ph1) {
    constexpr uint32_t size = 1u << K;
#pragma unroll(K < kLsegUnrollK ? (1 << K) : 4)
    for (uint32_t j = 0; j < size; j++) {
      const double2 v = arr[j];
      arr[j] = FS_SEG_CMUL(v, ph0);
      arr[size + j] = FS_SEG_CMUL(v, ph1);
    }
  }

  template <int AX, int K>
  __device__ __forceinline__ void array_rot(double2 ph0, double2 ph1) {
    constexpr uint32_t size = 1u << K;
#pragma unroll(K <= kLsegUnrollK ? (1 << K) : 4)
    for (uint32_t j = 0; j < size; j++) arr[j] = FS_SEG_CMUL(arr[j], ((j >> AX) & 1) ? ph1 : ph0);
  }

  // MeasActive / MeasCollapse (runtime.py:409-511; the interpreter's lane-per-shot form): false
  // when the shot stopped (NaN)
  template <bool COLLAPSE, int AX, int K>
  __device__ __forceinline__ bool measure(int i, int xv, int flip, int col, int sl, double2 u00, double2 u01,
                                          double2 u10, double2 u11) {
    constexpr uint32_t size = 1u << K, half = size >> 1, st = 1u << AX;
    double p1 = 0.0, p_all = 0.0;
#pragma unroll(K <= kLsegUnrollK ? (1 << K) : 4)
    for (uint32_t j = 0; j < half; j++) {
      const uint32_t i0 = ins0(j, AX);
      const double2 a0 = arr[i0], a1 = arr[i0 + st];
      if (COLLAPSE) p1 = __dadd_rn(p1, cnorm2(cadd(FS_SEG_CMUL(a0, u10), FS_SEG_CMUL(u11, a1))));
      else p1 = __dadd_rn(p1, cnorm2(a1));
      p_all = __dadd_rn(p_all, __dadd_rn(cnorm2(a0), cnorm2(a1)));
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
      // in place, ascending: element j reads ins0(j) >= j and ins0(j) + st > j only
#pragma unroll(K <= kLsegUnrollK ? (1 << K) : 4)
      for (uint32_t j = 0; j < half; j++) {
        const uint32_t i0 = ins0(j, AX);
        arr[j] = cadd(FS_SEG_CMUL(k0, arr[i0]), FS_SEG_CMUL(k1, arr[i0 + st]));
      }
    } else {
      const double s = renorm ? __ddiv_rn(1.0, __dsqrt_rn(pb)) : 1.0;
      const uint32_t dead = 1u - (uint32_t)br;
#pragma unroll(K <= kLsegUnrollK ? (1 << K) : 4)
      for (uint32_t j = 0; j < size; j++) {
        if (((j >> AX) & 1) == dead) arr[j] = make_double2(0.0, 0.0);
        else if (renorm) arr[j] = cscale(arr[j], s);
      }
    }
    return true;
  }

  template <int AX, int K>
  __device__ __forceinline__ void retire(int xv) {
    constexpr uint32_t half = (1u << K) >> 1;
    if (K <= kLsegUnrollK) {  // constant indices only: pick by the branch bit
#pragma unroll
      for (uint32_t j = 0; j < half; j++) {
        const double2 v0 = arr[ins0(j, AX)], v1 = arr[ins0(j, AX) + (1u << AX)];
        arr[j] = branch ? v1 : v0;
      }
    } else {
#pragma unroll 4
      for (uint32_t j = 0; j < half; j++) arr[j] = arr[ins0(j, AX) + ((uint32_t)branch << AX)];
    }
    fxor(xv, (uint32_t)branch);
  }
};

// the shot loop of a specialised lane-per-shot segment: array of 2^KIN in, 2^KOUT out, the last
// NLAZY Expands (2^(KOUT - NLAZY) -> 2^KOUT) folded into the save
template <int KARR, int KIN, int KOUT, int NLAZY, class Exec>
__device__ __forceinline__ void lseg_run(const DevProg& P, const RunArgs& A, const SegArgs& S, Exec&& exec) {
  const int lane = threadIdx.x & 31;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const uint32_t n_pad = (S.n_in + 31u) & ~31u;  // whole warps reach the compaction
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n_pad; idx += nthreads) {
    bool valid = idx < S.n_in;
    const uint64_t si = S.first ? S.chunk0 + idx : (valid ? S.in.shot[idx] : 0);
    valid = valid && si < A.nshots;
    double2 arr[1 << KARR];
    LCtx<KARR, NLAZY> c(P, A, S, si, arr);
    double2 gamma = make_double2(1.0, 0.0);
    if (valid) {
      if (S.first) {
        c.arr[0] = make_double2(1.0, 0.0);
      } else {
        const StateStore& I = S.in;
        c.load_scalars(I, idx);
        gamma = I.gamma[idx];
        const double2* const src = I.amps + store_amp_index(idx, 0, 1u << KIN, I.shot_major);
        const uint32_t sstride = I.shot_major ? 1u : 32u;
#pragma unroll(KIN <= kLsegUnrollK ? (1 << KIN) : 4)
        for (uint32_t j = 0; j < (1u << KIN); j++) c.arr[j] = src[(size_t)j * sstride];
      }
      exec(c);
    }
    __syncwarp();
    const bool alive = valid && c.alive != 0, errored = c.err != 0;
    if (valid && errored) {
      atomicOr(A.error + (si >> 5), 1u << (si & 31));
      atomicMax(A.status, c.err);
    }
    if (valid && (S.last || !alive)) {
      for (int o = 0; o < P.O; o++)
        if ((c.obs >> o) & 1u) c.out_bit(A.obs + (size_t)o * A.W);
      if (alive && !errored) c.out_bit(A.accepted);
    }
    if (!S.last) {  // survivors: compact into the output store
      const uint32_t surv = __ballot_sync(0xFFFFFFFFu, alive);
      uint32_t base = 0;
      if (lane == 0 && surv) base = atomicAdd(S.n_out, (uint32_t)__popc(surv));
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (alive) {
        c.settle_pending();
        const uint32_t slot = base + (uint32_t)__popc(surv & ((1u << lane) - 1u));
        const StateStore& O = S.out;
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (k < S.nfw) O.frame[(size_t)slot * S.nfw + k] = c.F[k];
        if (S.nsw) O.slotbits[(size_t)slot * S.nsw] = c.slots;
        if (S.now) O.obsbits[(size_t)slot * S.now] = c.obs;
        O.shot[slot] = (uint32_t)si;
        O.gamma[slot] = gamma;
        uint32_t* gi = O.gen_i + (size_t)slot * 6;
        gi[0] = c.gen.step_no; gi[1] = (uint32_t)c.gen.run; gi[2] = (uint32_t)c.gen.cl;
        gi[3] = (uint32_t)c.pend_site; gi[4] = (uint32_t)c.pend_lane; gi[5] = (uint32_t)c.pend_case;
        O.gen_c[slot] = c.gen.c;
        constexpr int KB = KOUT - NLAZY;  // array held at the save
        double2* const dst = O.amps + store_amp_index(slot, 0, 1u << KOUT, O.shot_major);
        const uint32_t dstride = O.shot_major ? 1u : 32u;
#pragma unroll(KOUT <= kLsegUnrollK ? (1 << NLAZY) : 1)
        for (uint32_t hi = 0; hi < (1u << NLAZY); hi++) {
#pragma unroll(KOUT <= kLsegUnrollK ? (1 << KB) : 4)
          for (uint32_t j = 0; j < (1u << KB); j++) {
            double2 v = c.arr[j];
#pragma unroll
            for (int t = 0; t < NLAZY; t++) v = FS_SEG_CMUL(v, ((hi >> t) & 1u) ? c.lz1[t] : c.lz0[t]);
            dst[(size_t)(j | (hi << KB)) * dstride] = v;
          }
        }
      }
    }
  }
}

}  // namespace fs
