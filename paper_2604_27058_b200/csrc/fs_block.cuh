// fs_block.cuh -- CTA-per-shot engine for segments whose active array is too large for a lane
// (2^k >= 64 amplitudes): the array of one shot lives in shared memory and every sweep is split
// across the CTA's threads; the scalar VM (frame bits, records, draws) runs on thread 0.
//
// Used by the segmented driver (post-selected programs, config 4): the survivor state store
// (fs_general.cuh StateStore) is engine-neutral, so consecutive segments may alternate between
// the lane-per-shot general engine (small k, many shots) and this engine (large k, few shots).
#pragma once
#include "fs_general.cuh"

namespace fs {

// G threads per shot: G = 32 (warp per shot, several shots per CTA) or G = 256 (CTA per shot)
constexpr int kBlockMaxGroups = 16;  // warp-per-shot groups per CTA (bounded by shared memory)

template <bool SPLITMIX, int G>
__global__ void __launch_bounds__(G == 32 ? 32 * kBlockMaxGroups : 256, G == 32 ? 2 : 4) block_kernel(DevProg P, RunArgs A, SegArgs S, int karr, int group_bytes) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t cap = 1u << karr;
  const int group = threadIdx.x / G, ngroups = blockDim.x / G;
  double2* amp = reinterpret_cast<double2*>(smem_raw + (size_t)group * group_bytes);
  uint32_t* fx = reinterpret_cast<uint32_t*>(amp + cap);  // one shot: values 0/1
  uint32_t* fz = fx + P.n;
  uint32_t* slots = fz + P.n;
  uint32_t* obsb = slots + P.num_slots;
  // reduction scratch only for the CTA-per-shot form (warp groups reduce with shuffles)
  __shared__ double red1s[G == 256 ? 256 : 1], red2s[G == 256 ? 256 : 1];
  __shared__ double2 sh_k0s[kBlockMaxGroups], sh_k1s[kBlockMaxGroups];
  __shared__ int sh_alives[kBlockMaxGroups], sh_branchs[kBlockMaxGroups], sh_errs[kBlockMaxGroups];
  __shared__ uint32_t sh_slots[kBlockMaxGroups];
  double2& sh_k0 = sh_k0s[group];
  double2& sh_k1 = sh_k1s[group];
  int& sh_alive = sh_alives[group];
  int& sh_branch = sh_branchs[group];
  int& sh_err = sh_errs[group];
  double* red1 = red1s;
  double* red2 = red2s;
  const int tid = threadIdx.x % G, nt = G;
  const bool renorm = !(A.flags & FS_NO_RENORM);
#define FS_BAR() do { if (G == 32) __syncwarp(); else __syncthreads(); } while (0)

  for (uint32_t idx = blockIdx.x * ngroups + group; idx < S.n_in; idx += gridDim.x * ngroups) {
    const uint64_t si = S.first ? S.chunk0 + idx : S.in.shot[idx];
    if (si >= A.nshots) continue;  // uniform over the block
    const uint64_t shot = A.shot0 + si;
    const uint64_t wabs = shot >> 5;
    const int mylane = (int)(shot & 31);
    // thread-0 scalar state
    double2 gamma = make_double2(1.0, 0.0);
    SplitMix sm;
    WordFaultGen gen;
    int pend_site = -1, pend_lane = 0, pend_case = 0;
    int branch = 0;
    int coin_blk = -1;  // thread 0: Philox coin block of ordinals 4b..4b+3, reused across coins
    uint4 coin_b = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
      sh_alive = 1;
      sh_err = 0;
      if (SPLITMIX) sm.reset(A.seed, shot);
      else gen.init(A.seed, wabs);
    }
    if (S.first) {
      for (int q = tid; q < 2 * P.n + P.num_slots + P.O; q += nt) fx[q] = 0;
      if (tid == 0) amp[0] = make_double2(1.0, 0.0);
    } else {
      const StateStore& I = S.in;
      for (int b = tid; b < 2 * P.n; b += nt)
        fx[b] = (I.frame[(size_t)idx * S.nfw + (b >> 5)] >> (b & 31)) & 1u;  // fz = fx + n
      for (int b = tid; b < P.num_slots; b += nt) slots[b] = (I.slotbits[(size_t)idx * S.nsw + (b >> 5)] >> (b & 31)) & 1u;
      for (int b = tid; b < P.O; b += nt) obsb[b] = (I.obsbits[(size_t)idx * S.now + (b >> 5)] >> (b & 31)) & 1u;
      const uint32_t sz = 1u << S.k_in, icap = 1u << S.k_in;
      for (uint32_t j = tid; j < sz; j += nt) amp[j] = I.amps[store_amp_index(idx, j, icap, I.shot_major)];
      if (tid == 0) {
        gamma = I.gamma[idx];
        if (SPLITMIX) sm.count = I.smcount[idx];
        else {
          gen.step_no = I.gen_i[(size_t)idx * 6];
          gen.run = (int)I.gen_i[(size_t)idx * 6 + 1];
          gen.cl = (int)I.gen_i[(size_t)idx * 6 + 2];
          pend_site = (int)I.gen_i[(size_t)idx * 6 + 3];
          pend_lane = (int)I.gen_i[(size_t)idx * 6 + 4];
          pend_case = (int)I.gen_i[(size_t)idx * 6 + 5];
          gen.c = I.gen_c[idx];
        }
      }
    }
    FS_BAR();
    auto out_bit = [&](uint32_t* row) { atomicOr(row + (si >> 5), 1u << (si & 31)); };
    // one scalar instruction of this shot (thread 0 only)
    auto scalar_step = [&](int i) {
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
          uint32_t bit;
          if (op == FS_OP_MEAS_DSTATIC) {
            bit = fx[virt] ^ (uint32_t)flip;
          } else {
            const uint32_t pz = fz[virt];
            uint32_t coin;
            if (SPLITMIX) {
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
          const int col = __ldg(P.record_out + rec);
          if (col >= 0 && bit) out_bit(A.meas + (size_t)col * A.W);
          const int sl = __ldg(P.bit_slot + rec);
          if (sl >= 0) slots[sl] = bit;
          break;
        }
        case FS_OP_COND_FRAME:
          if (slots[__ldg(P.bit_slot + ins[3])]) xor_paulis<false>(P, fx, fz, ins[1], ins[2], 1u);
          break;
        case FS_OP_NOISE:
          if (SPLITMIX) {
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
          if ((int)slots[__ldg(P.bit_slot + bid)] != ins[3]) sh_alive = 0;
          break;
        }
        default: break;
      }
    };
    for (int i = S.seg_begin; i < S.seg_end; i++) {
      if (!sh_alive) break;
      {  // a run of scalar instructions executes on thread 0 with one barrier at its end
        const int j = min(__ldg(P.next_array + i), S.seg_end);
        if (j > i) {
          if (tid == 0)
            for (int t = i; t < j && sh_alive; t++) scalar_step(t);
          FS_BAR();
          i = j - 1;
          continue;
        }
      }
      const int4 I0 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i);
      const int4 I1 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i + 1);
      const int ins[8] = {I0.x, I0.y, I0.z, I0.w, I1.x, I1.y, I1.z, I1.w};
      const int op = FS_OPCODE(I0.x);
      const int flip = FS_FLIP(I0.x);
      switch (op) {
        case FS_OP_FRAME: {  // GF(2) matrix (next_array stops here only when it exists)
          const int mo = __ldg(P.frame_mat_off + i);
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
          FS_BAR();
          break;
        }
        case FS_OP_ARRAY_GATE: {
          const int g = ins[1], va = ins[2], vb = ins[3], a = ins[4], b = ins[5];
          const uint32_t size = 1u << ins[6];
          if (g == FS_G_S || g == FS_G_SDAG) {
            const double2 ph = make_double2(0.0, g == FS_G_S ? 1.0 : -1.0);
            for (uint32_t j = tid; j < size / 2; j += nt) {
              const uint32_t id = ins0(j, a) | (1u << a);
              amp[id] = cmul(amp[id], ph);
            }
          } else if (g == FS_G_H) {
            const uint32_t st = 1u << a;
            for (uint32_t j = tid; j < size / 2; j += nt) {
              const uint32_t i0 = ins0(j, a);
              const double2 lo = amp[i0], hi = amp[i0 + st];
              amp[i0] = cscale(cadd(lo, hi), kInvSqrt2);
              amp[i0 + st] = cscale(csub(lo, hi), kInvSqrt2);
            }
          } else {
            const int lo_ax = a < b ? a : b, hi_ax = a < b ? b : a;
            for (uint32_t j = tid; j < size / 4; j += nt) {
              const uint32_t id = ins0(ins0(j, lo_ax), hi_ax) | (1u << a);
              if (g == FS_G_CX) {
                const uint32_t jd = id | (1u << b);
                const double2 t0 = amp[id];
                amp[id] = amp[jd];
                amp[jd] = t0;
              } else {
                const uint32_t jd = id | (1u << b);
                const double2 v = amp[jd];
                amp[jd] = make_double2(-v.x, -v.y);
              }
            }
          }
          if (tid == 0) {
            uint32_t t;
            switch (g) {
              case FS_G_S: case FS_G_SDAG: fz[va] ^= fx[va]; break;
              case FS_G_H: t = fx[va]; fx[va] = fz[va]; fz[va] = t; break;
              case FS_G_CX: fx[vb] ^= fx[va]; fz[va] ^= fz[vb]; break;
              case FS_G_CZ: fz[vb] ^= fx[va]; fz[va] ^= fx[vb]; break;
            }
          }
          FS_BAR();
          break;
        }
        case FS_OP_EXPAND: {
          const int par = fx[ins[1]] & 1;
          const double* f = P.fparams + ins[5] + 4 * par;
          const double2 ph0 = make_double2(__ldg(f), __ldg(f + 1)), ph1 = make_double2(__ldg(f + 2), __ldg(f + 3));
          const uint32_t size = 1u << ins[6];
          for (uint32_t j = tid; j < size; j += nt) {
            const double2 v = amp[j];
            amp[j] = cmul(v, ph0);
            amp[size + j] = cmul(v, ph1);
          }
          FS_BAR();
          break;
        }
        case FS_OP_ARRAY_ROT: {
          const int par = fx[ins[1]] & 1, a = ins[2];
          const double* f = P.fparams + ins[5];
          const double2 e0 = make_double2(__ldg(f), __ldg(f + 1)), e1 = make_double2(__ldg(f + 2), __ldg(f + 3));
          const double2 ph0 = par ? e1 : e0, ph1 = par ? e0 : e1;
          const uint32_t size = 1u << ins[6];
          for (uint32_t j = tid; j < size; j += nt) amp[j] = cmul(amp[j], ((j >> a) & 1) ? ph1 : ph0);
          FS_BAR();
          break;
        }
        case FS_OP_MEAS_ACTIVE:
        case FS_OP_MEAS_COLLAPSE: {
          const int virt = ins[1], a = ins[2], rec = ins[3];
          const uint32_t size = 1u << ins[6], half = size >> 1, st = 1u << a;
          const bool collapse = op == FS_OP_MEAS_COLLAPSE;
          double2 u00 = make_double2(1, 0), u01 = make_double2(0, 0), u10 = make_double2(0, 0), u11 = make_double2(1, 0);
          if (collapse) {
            const double* f = P.fparams + ins[5];
            u00 = make_double2(__ldg(f), __ldg(f + 1));
            u01 = make_double2(__ldg(f + 2), __ldg(f + 3));
            u10 = make_double2(__ldg(f + 4), __ldg(f + 5));
            u11 = make_double2(__ldg(f + 6), __ldg(f + 7));
          }
          // (p1, p_all) partial sums in a fixed order per thread, then a fixed-order tree
          double s1 = 0.0, sa = 0.0;
          for (uint32_t j = tid; j < half; j += nt) {
            const uint32_t i0 = ins0(j, a);
            const double2 a0 = amp[i0], a1 = amp[i0 + st];
            if (collapse) {
              s1 = __dadd_rn(s1, cnorm2(cadd(cmul(a0, u10), cmul(u11, a1))));
            } else {
              s1 = __dadd_rn(s1, cnorm2(a1));
            }
            sa = __dadd_rn(sa, __dadd_rn(cnorm2(a0), cnorm2(a1)));
          }
          // fixed-order tree: element t += element t + w for w = nt/2 .. 1 (same pairs either way)
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
            FS_BAR();
            for (int w = nt >> 1; w; w >>= 1) {
              if (tid < w) {
                red1[tid] = __dadd_rn(red1[tid], red1[tid + w]);
                red2[tid] = __dadd_rn(red2[tid], red2[tid + w]);
              }
              FS_BAR();
            }
            s1 = red1[0];
            sa = red2[0];
          }
          if (tid == 0) {
            if (collapse) {
              const int po = ins[4] >> 8, pc = ins[4] & 0xFF;
              for (int j = 0; j < pc; j++) word_gate(fx, fz, __ldg(P.gates + po + j));
            }
            double p1 = s1, p_all = sa;
            const int parity = fx[virt] & 1;
            int bad = 0;
            if (p1 != p1) bad = FS_ERR_SHOT_NAN;
            if (collapse || !renorm) p1 = p_all > 0 ? __ddiv_rn(p1, p_all) : 0.0;
            if (p1 < 0.0) p1 = 0.0;
            else if (p1 > 1.0) p1 = 1.0;
            double u;
            if (SPLITMIX) u = sm.uniform();
            else {
              const uint4 o = philox((uint32_t)shot, (uint32_t)(shot >> 32), (uint32_t)i, TAG_BORN << 24, A.seed);
              u = u64_to_unit(((uint64_t)o.y << 32) | o.x);
            }
            int br = u < p1 ? 1 : 0;
            double pb = br ? p1 : __dsub_rn(1.0, p1);
            if (pb < kBranchFloor) { br ^= 1; pb = __dsub_rn(1.0, pb); }
            if (bad) {
              sh_err = bad;
              sh_alive = 0;
            } else {
              const uint32_t recbit = (uint32_t)(br ^ parity ^ flip);
              const int col = __ldg(P.record_out + rec);
              if (col >= 0 && recbit) out_bit(A.meas + (size_t)col * A.W);
              const int sl = __ldg(P.bit_slot + rec);
              if (sl >= 0) slots[sl] = recbit;
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
          FS_BAR();
          if (!sh_alive) break;
          branch = sh_branch;
          if (collapse) {  // compaction: gather sources first (in-place, different threads)
            const double2 k0 = sh_k0, k1 = sh_k1;
            // in place, one strip of nt outputs at a time: strip b reads indices >= its own
            // outputs, all above what earlier strips wrote
            for (uint32_t b0 = 0; b0 < half; b0 += nt) {
              const uint32_t j = b0 + tid;
              double2 val = make_double2(0.0, 0.0);
              if (j < half) {
                const uint32_t i0 = ins0(j, a);
                val = cadd(cmul(k0, amp[i0]), cmul(k1, amp[i0 + st]));
              }
              FS_BAR();
              if (j < half) amp[j] = val;
              FS_BAR();
            }
          } else {
            const double s = sh_k0.x;
            const uint32_t dead = 1u - (uint32_t)branch;
            for (uint32_t j = tid; j < size; j += nt) {
              if (((j >> a) & 1) == dead) amp[j] = make_double2(0.0, 0.0);
              else if (renorm) amp[j] = cscale(amp[j], s);
            }
          }
          FS_BAR();
          break;
        }
        case FS_OP_RETIRE: {
          const int virt = ins[1], a = ins[2];
          const uint32_t half = (1u << ins[6]) >> 1;
          const int br = sh_branch;
          for (uint32_t b0 = 0; b0 < half; b0 += nt) {  // in place, strip by strip (as collapse)
            const uint32_t j = b0 + tid;
            double2 val = make_double2(0.0, 0.0);
            if (j < half) val = amp[ins0(j, a) + ((uint32_t)br << a)];
            FS_BAR();
            if (j < half) amp[j] = val;
            FS_BAR();
          }
          if (tid == 0) fx[virt] ^= (uint32_t)br;
          FS_BAR();
          break;
        }
        default:
          break;
      }
    }
    FS_BAR();
    const bool alive = sh_alive != 0;
    const bool errored = sh_err != 0;
    if (tid == 0) {
      if (errored) {
        atomicOr(A.error + (si >> 5), 1u << (si & 31));
        atomicMax(A.status, sh_err);
      }
      if (S.last || !alive) {
        for (int o = 0; o < P.O; o++)
          if (obsb[o]) out_bit(A.obs + (size_t)o * A.W);
        if (alive && !errored) out_bit(A.accepted);
      }
    }
    if (!S.last && alive) {  // survivor: compact into the output store
      if (tid == 0) sh_slots[group] = atomicAdd(S.n_out, 1u);
      FS_BAR();
      const uint32_t slot = sh_slots[group];
      const StateStore& O = S.out;
      for (int j = tid; j < S.nfw; j += nt) {
        uint32_t v = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < 2 * P.n; b++) v |= (fx[b] & 1u) << (b & 31);
        O.frame[(size_t)slot * S.nfw + j] = v;
      }
      for (int j = tid; j < S.nsw; j += nt) {
        uint32_t v = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < P.num_slots; b++) v |= (slots[b] & 1u) << (b & 31);
        O.slotbits[(size_t)slot * S.nsw + j] = v;
      }
      for (int j = tid; j < S.now; j += nt) {
        uint32_t v = 0;
        for (int b = 32 * j; b < 32 * j + 32 && b < P.O; b++) v |= (obsb[b] & 1u) << (b & 31);
        O.obsbits[(size_t)slot * S.now + j] = v;
      }
      const uint32_t sz = 1u << S.k_out;
      for (uint32_t j = tid; j < sz; j += nt) O.amps[store_amp_index(slot, j, sz, O.shot_major)] = amp[j];
      if (tid == 0) {
        O.shot[slot] = (uint32_t)si;
        O.gamma[slot] = gamma;
        if (SPLITMIX) O.smcount[slot] = sm.count;
        else {
          uint32_t* gi = O.gen_i + (size_t)slot * 6;
          gi[0] = gen.step_no; gi[1] = (uint32_t)gen.run; gi[2] = (uint32_t)gen.cl;
          gi[3] = (uint32_t)pend_site; gi[4] = (uint32_t)pend_lane; gi[5] = (uint32_t)pend_case;
          O.gen_c[slot] = gen.c;
        }
      }
    }
    FS_BAR();
  }
#undef FS_BAR
}

}  // namespace fs
