// fs_hbm.cuh -- the large-k engine: active arrays resident in HBM, whole GPU per instruction.
//
// Used when 32 * 2^k_max complex128 per warp cannot live on chip (k_max >= 16, e.g. config 3
// at k = 22: 64 MiB per shot).  A batch of B shots is processed together:
//
//   * scalar kernel (thread = 32-shot word, bit-sliced frames kept in HBM between launches)
//     executes every non-array instruction and the frame side of array instructions, records
//     the frame-parity word each Expand / ArrayRot needs (par[instr][word]) and takes the
//     measurement decisions once the array reduction is available;
//   * array kernels sweep B x 2^k amplitudes per array instruction, touching only the
//     elements the instruction changes (CZ: 1/4, CX/S: 1/2, ...);
//   * measurement: deterministic two-level reduction of (p1, p_all) per shot, then the scalar
//     kernel draws the branch, then an in-place collapse.
//
// Physical layout: arrays never move after a measurement.  The host keeps a logical->physical
// axis map; a collapse writes k0*a0 + k1*a1 into the bit-0 position of the measured physical
// axis, which then becomes "dead" (all valid elements have it 0) and is reused by a later
// Expand.  Every kernel enumerates the 2^k valid elements by inserting zero bits at the dead
// physical positions, so all updates are in place and race-free.
#pragma once
#include "fs_general.cuh"

namespace fs {

constexpr int kHbmMaxDead = 32;

struct DevAxisMap {
  int8_t phys[32];  // logical axis -> physical bit position
};

// logical element counter -> physical index: insert a 0 bit at every listed position (ascending;
// the list = dead physical axes below the top live one plus the op's own axes)
struct DeadBits {
  int n;
  int8_t pos[kHbmMaxDead];
  __device__ __forceinline__ uint64_t expand(uint64_t j) const {
    for (int d = 0; d < n; d++) {
      const int p = pos[d];
      const uint64_t low = j & ((1ull << p) - 1ull);
      j = ((j - low) << 1) | low;
    }
    return j;
  }
};

struct HbmState {
  uint32_t* fx;       // [n][W]
  uint32_t* fz;       // [n][W]
  uint32_t* slots;    // [S][W]
  uint32_t* obs;      // [O][W]
  uint32_t* alive;    // [W]
  uint32_t* err;      // [W]
  uint32_t* par;      // [N][W] parity words for Expand / ArrayRot
  uint32_t* brw;      // [W]   branch word of the current measurement
  uint32_t* frozen;   // [W]   shots whose trace frames were written at their halt point
  double2* gamma;     // [B]
  uint32_t* smcount;  // [B]   SplitMix draw counters
  double* red;        // [B][2*nblk] partial (p1, p_all)
  double* p1;         // [B]
  double* pall;       // [B]
  double2* kco;       // [B][2] collapse coefficients
  double2* amps;      // [B][cap]
  uint64_t cap;
  int nblk;           // reduction blocks per shot
  int errcode_dummy;
};

// ------------------------------------------------------------------ scalar kernel
// Executes instructions [i0, i1) for every word of the batch.  If `meas` >= 0 instruction i0
// is that measurement and its (p1, p_all) reduction is ready.
template <bool SPLITMIX>
__global__ void __launch_bounds__(128) hbm_scalar_kernel(DevProg P, RunArgs A, HbmState H, int i0, int i1,
                                                           int init, uint64_t batch0, uint32_t W) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;  // word within the batch
  if (w >= W) return;
  const uint64_t si0 = batch0 + (uint64_t)w * 32;  // shot index (within the call) of bit 0
  const uint64_t nleft = A.nshots - si0;
  const uint32_t validmask = nleft >= 32 ? kFull : ((1u << nleft) - 1u);
  const uint32_t gw = (uint32_t)(si0 >> 5);         // output word
  const uint64_t wabs = (A.shot0 >> 5) + gw;
  const bool renorm = !(A.flags & FS_NO_RENORM);
  uint32_t* fx = H.fx + w;
  uint32_t* fz = H.fz + w;
  uint32_t* slots = H.slots + w;
  // stride between qubits / slots = W (column-major words)
#define FX(q) fx[(size_t)(q) * W]
#define FZ(q) fz[(size_t)(q) * W]
#define SL(s) slots[(size_t)(s) * W]
  if (init) {
    for (int q = 0; q < P.n; q++) { FX(q) = 0; FZ(q) = 0; }
    for (int o = 0; o < P.O; o++) H.obs[(size_t)o * W + w] = 0;
    H.alive[w] = validmask;
    H.err[w] = 0;
    H.frozen[w] = 0;
    for (int j = 0; j < 32; j++) {
      const uint64_t bs = (uint64_t)w * 32 + j;  // shot within the batch
      if (!((validmask >> j) & 1)) continue;
      H.gamma[bs] = make_double2(1.0, 0.0);
      H.smcount[bs] = A.draw0 ? A.draw0[si0 + j] : 0u;
    }
  }
  uint32_t alive = H.alive[w];
  uint32_t errmask = H.err[w];
  int errcode = 0;
  for (int i = i0; i < i1; i++) {
    if (alive == 0) break;
    const int4 I0 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i);
    const int4 I1 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i + 1);
    const int ins[8] = {I0.x, I0.y, I0.z, I0.w, I1.x, I1.y, I1.z, I1.w};
    const int op = FS_OPCODE(I0.x);
    const int flip = FS_FLIP(I0.x);
    const uint32_t flipw = flip ? kFull : 0u;
    switch (op) {
      case FS_OP_FRAME:
        for (int j = 0; j < ins[2]; j++) {
          uint32_t g = __ldg(P.gates + ins[1] + j);
          int a = FS_GATE_A(g), b = FS_GATE_B(g);
          uint32_t t;
          switch (FS_GATE_G(g)) {
            case FS_G_H: t = FX(a); FX(a) = FZ(a); FZ(a) = t; break;
            case FS_G_S: case FS_G_SDAG: FZ(a) ^= FX(a); break;
            case FS_G_CX: FX(b) ^= FX(a); FZ(a) ^= FZ(b); break;
            case FS_G_CZ: FZ(b) ^= FX(a); FZ(a) ^= FX(b); break;
            case FS_G_SWAP: t = FX(a); FX(a) = FX(b); FX(b) = t; t = FZ(a); FZ(a) = FZ(b); FZ(b) = t; break;
          }
        }
        break;
      case FS_OP_ARRAY_GATE: {
        const int g = ins[1], va = ins[2], vb = ins[3];
        uint32_t t;
        switch (g) {
          case FS_G_S: case FS_G_SDAG: FZ(va) ^= FX(va); break;
          case FS_G_H: t = FX(va); FX(va) = FZ(va); FZ(va) = t; break;
          case FS_G_CX: FX(vb) ^= FX(va); FZ(va) ^= FZ(vb); break;
          case FS_G_CZ: FZ(vb) ^= FX(va); FZ(va) ^= FX(vb); break;
        }
        break;
      }
      case FS_OP_EXPAND:
      case FS_OP_ARRAY_ROT:
        H.par[(size_t)i * W + w] = FX(ins[1]);
        break;
      case FS_OP_GAMMA_ROT: {
        const uint32_t pw = FX(ins[1]);
        const double* f = P.fparams + ins[5];
        for (int j = 0; j < 32; j++) {
          if (!((alive >> j) & 1)) continue;
          const int par = (pw >> j) & 1;
          const uint64_t bs = (uint64_t)w * 32 + j;
          H.gamma[bs] = cmul(H.gamma[bs], make_double2(__ldg(f + 2 * par), __ldg(f + 2 * par + 1)));
        }
        break;
      }
      case FS_OP_RETIRE: {  // branch word of the preceding MeasActive
        FX(ins[1]) ^= H.brw[w] & alive;
        break;
      }
      case FS_OP_MEAS_DSTATIC:
      case FS_OP_MEAS_DRANDOM: {
        const int virt = ins[1], rec = ins[3];
        uint32_t recw;
        if (op == FS_OP_MEAS_DSTATIC) {
          recw = FX(virt) ^ flipw;
          if (A.forced) {
            uint32_t bad = 0;
            for (int j = 0; j < 32; j++) {
              if (!((alive >> j) & 1)) continue;
              int fo = A.forced[(si0 + j) * P.R + rec];
              if (fo >= 0 && fo != (int)((recw >> j) & 1)) bad |= 1u << j;
            }
            if (bad) { errmask |= bad; alive &= ~bad; errcode = FS_ERR_SHOT_FORCED; }
          }
        } else {
          const uint32_t pw = FZ(virt);
          uint32_t coinw = 0;
          if (!SPLITMIX) coinw = coin_word(A.seed, wabs, ins[2]);
          for (int j = 0; j < 32; j++) {
            if (!((validmask >> j) & 1)) continue;
            const int fo = A.forced ? A.forced[(si0 + j) * P.R + rec] : -1;
            uint32_t c;
            if (fo >= 0) c = (uint32_t)(fo ^ (int)((pw >> j) & 1) ^ flip);
            else if (SPLITMIX) {
              if (!((alive >> j) & 1)) { c = 0; }
              else {
                const uint64_t bs = (uint64_t)w * 32 + j;
                SplitMix sm;
                sm.key = mix64(mix64(A.seed) ^ (A.shot0 + si0 + j));
                sm.count = H.smcount[bs];
                c = (uint32_t)sm.bit();
                H.smcount[bs] = sm.count;
              }
            } else c = (coinw >> j) & 1;
            coinw = (coinw & ~(1u << j)) | (c << j);
          }
          const uint32_t t = FX(virt);
          FX(virt) = FZ(virt) ^ coinw;
          FZ(virt) = t;
          for (int j = 0; j < 32; j++) {
            if (!((alive >> j) & 1)) continue;
            const uint64_t bs = (uint64_t)w * 32 + j;
            H.gamma[bs] = cscale(H.gamma[bs], kInvSqrt2);
          }
          recw = coinw ^ pw ^ flipw;
        }
        const int col = __ldg(P.record_out + rec);
        if (col >= 0) A.meas[(size_t)col * A.W + gw] = recw & alive;
        const int sl = __ldg(P.bit_slot + rec);
        if (sl >= 0) SL(sl) = recw;
        if (A.t_rec)
          for (int b = 0; b < 32; b++)
            if ((alive >> b) & 1) A.t_rec[(si0 + b) * P.R + rec] = (uint8_t)((recw >> b) & 1);
        break;
      }
      case FS_OP_MEAS_ACTIVE:
      case FS_OP_MEAS_COLLAPSE: {
        // decision half (the reduction ran before this launch; the collapse runs after it)
        const int virt = ins[1], rec = ins[3];
        const bool collapse = op == FS_OP_MEAS_COLLAPSE;
        if (collapse) {
          const int po = ins[4] >> 8, pc = ins[4] & 0xFF;
          for (int j = 0; j < pc; j++) {
            uint32_t g = __ldg(P.gates + po + j);
            int a = FS_GATE_A(g);
            if (FS_GATE_G(g) == FS_G_H) { uint32_t t = FX(a); FX(a) = FZ(a); FZ(a) = t; }
            else FZ(a) ^= FX(a);
          }
        }
        const uint32_t pxw = FX(virt);
        uint32_t recw = 0, brw = 0, bad = 0;
        int badcode = 0;
        double2 u00 = make_double2(1, 0), u01 = make_double2(0, 0), u10 = make_double2(0, 0), u11 = make_double2(1, 0);
        if (collapse) {
          const double* f = P.fparams + ins[5];
          u00 = make_double2(__ldg(f), __ldg(f + 1));
          u01 = make_double2(__ldg(f + 2), __ldg(f + 3));
          u10 = make_double2(__ldg(f + 4), __ldg(f + 5));
          u11 = make_double2(__ldg(f + 6), __ldg(f + 7));
        }
        for (int j = 0; j < 32; j++) {
          if (!((alive >> j) & 1)) continue;
          const uint64_t bs = (uint64_t)w * 32 + j;
          const int parity = (pxw >> j) & 1;
          double p1 = H.p1[bs], p_all = H.pall[bs];
          if (p1 != p1) { bad |= 1u << j; badcode = FS_ERR_SHOT_NAN; continue; }
          if (collapse) p1 = p_all > 0 ? __ddiv_rn(p1, p_all) : 0.0;
          else if (!renorm) p1 = p_all > 0 ? __ddiv_rn(p1, p_all) : 0.0;
          if (p1 < 0.0) p1 = 0.0;
          else if (p1 > 1.0) p1 = 1.0;
          const int fo = A.forced ? A.forced[(si0 + j) * P.R + rec] : -1;
          int br;
          double pb;
          if (fo < 0) {
            double u;
            if (SPLITMIX) {
              SplitMix sm;
              sm.key = mix64(mix64(A.seed) ^ (A.shot0 + si0 + j));
              sm.count = H.smcount[bs];
              u = sm.uniform();
              H.smcount[bs] = sm.count;
            } else {
              const uint64_t shot = A.shot0 + si0 + j;
              uint4 o = philox((uint32_t)shot, (uint32_t)(shot >> 32), (uint32_t)i, TAG_BORN << 24, A.seed);
              u = u64_to_unit(((uint64_t)o.y << 32) | o.x);
            }
            br = u < p1 ? 1 : 0;
            pb = br ? p1 : __dsub_rn(1.0, p1);
            if (pb < kBranchFloor) { br ^= 1; pb = __dsub_rn(1.0, pb); }
          } else {
            br = fo ^ parity ^ flip;
            pb = br ? p1 : __dsub_rn(1.0, p1);
            if (pb < kBranchFloor) { bad |= 1u << j; badcode = FS_ERR_SHOT_FORCED; continue; }
          }
          recw |= (uint32_t)(br ^ parity ^ flip) << j;
          brw |= (uint32_t)br << j;
          double2 k0, k1;
          if (collapse) {
            const double scale = renorm ? __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(pb, p_all))) : 1.0;
            k0 = br == 0 ? cscale(u00, scale) : cscale(u10, scale);
            k1 = br == 0 ? cscale(u01, scale) : cscale(u11, scale);
          } else {
            const double scale = renorm ? __ddiv_rn(1.0, __dsqrt_rn(pb)) : 1.0;
            k0 = make_double2(scale, 0.0);  // live-half scale
            k1 = make_double2(0.0, 0.0);
          }
          H.kco[2 * bs] = k0;
          H.kco[2 * bs + 1] = k1;
          if (renorm) H.gamma[bs] = cscale(H.gamma[bs], __dsqrt_rn(pb));
        }
        if (bad) { errmask |= bad; alive &= ~bad; errcode = badcode; }
        H.brw[w] = brw;
        if (collapse) FX(virt) ^= brw;
        const int col = __ldg(P.record_out + rec);
        if (col >= 0) A.meas[(size_t)col * A.W + gw] = recw & alive;
        const int sl = __ldg(P.bit_slot + rec);
        if (sl >= 0) SL(sl) = recw;
        if (A.t_rec)
          for (int b = 0; b < 32; b++)
            if ((alive >> b) & 1) A.t_rec[(si0 + b) * P.R + rec] = (uint8_t)((recw >> b) & 1);
        break;
      }
      case FS_OP_COND_FRAME: {
        const uint32_t rw = SL(__ldg(P.bit_slot + ins[3]));
        if (rw)
          for (int j = 0; j < ins[2]; j++) {
            uint32_t e = __ldg(P.paulis + ins[1] + j);
            if (FS_PAULI_Z(e)) FZ(FS_PAULI_Q(e)) ^= rw; else FX(FS_PAULI_Q(e)) ^= rw;
          }
        break;
      }
      case FS_OP_NOISE: {
        // frame words are strided by W: use the strided helpers on a W-stride view
        if (A.fault_modes || SPLITMIX) {
          for (int j = 0; j < 32; j++) {
            if (!((alive >> j) & 1)) continue;
            const uint64_t bs = (uint64_t)w * 32 + j;
            const uint64_t shot = A.shot0 + si0 + j;
            if (A.fault_modes) {
              ShotDraws d;
              d.splitmix = SPLITMIX;
              d.seed = A.seed;
              d.shot = shot;
              if (SPLITMIX) { d.sm.key = mix64(mix64(A.seed) ^ shot); d.sm.count = H.smcount[bs]; }
              d.begin(i, TAG_FORCED);
              forced_faults_shot(P, fx, fz, 1u << j, ins, A.fault_modes + (si0 + j) * P.E, d, (int)W);
              if (SPLITMIX) H.smcount[bs] = d.sm.count;
            } else {
              SplitMix sm;
              sm.key = mix64(mix64(A.seed) ^ shot);
              sm.count = H.smcount[bs];
              hazard_shot(P, fx, fz, 1u << j, ins, sm, (int)W, false);
              H.smcount[bs] = sm.count;
            }
          }
        } else {
          // the word's fault generator state persists in HBM between launches: regenerate
          // and skip the sites before this block (cheap: the HBM engine is array-bound)
          FaultBuffer<kFaultCap> fb;
          fb.init(P, A.seed, wabs);
          fb.apply_until(P, ins[1], [&](int, int) {});
          fb.apply_until(P, ins[2], [&](int c, int l) {
            const int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
            for (int jj = off; jj < end; jj++) {
              const uint32_t e = __ldg(P.paulis + jj);
              (FS_PAULI_Z(e) ? fz : fx)[(size_t)FS_PAULI_Q(e) * W] ^= 1u << l;
            }
          });
        }
        break;
      }
      case FS_OP_DETECTOR:
      case FS_OP_OBSERVABLE: {
        uint32_t wv = 0;
        for (int j = 0; j < ins[3]; j++) wv ^= SL(__ldg(P.bit_slot + __ldg(P.reclists + ins[2] + j)));
        if (op == FS_OP_DETECTOR) {
          A.det[(size_t)ins[1] * A.W + gw] = wv & alive;
          const int sl = __ldg(P.bit_slot + P.R + ins[1]);
          if (sl >= 0) SL(sl) = wv;
        } else {
          H.obs[(size_t)ins[1] * W + w] ^= wv & alive;
        }
        break;
      }
      case FS_OP_POSTSELECT: {
        const int bid = ins[1] == 0 ? P.R + ins[2] : ins[2];
        const uint32_t bw = SL(__ldg(P.bit_slot + bid));
        const uint32_t rej = (bw ^ (ins[3] ? kFull : 0u)) & alive;
        alive &= ~rej;
        if (rej && A.t_fx) {  // a rejected shot's frame freezes at its halt point
          for (int j = 0; j < 32; j++) {
            if (!((rej >> j) & 1)) continue;
            for (int q = 0; q < P.n; q++) {
              A.t_fx[(si0 + j) * P.n + q] = (FX(q) >> j) & 1;
              A.t_fz[(si0 + j) * P.n + q] = (FZ(q) >> j) & 1;
            }
          }
          H.frozen[w] |= rej;
        }
        break;
      }
      default: break;
    }
  }
  H.alive[w] = alive;
  H.err[w] = errmask;
  if (errcode) atomicMax(A.status, errcode);
#undef FX
#undef FZ
#undef SL
}

// finalisation of a batch: observables / accepted / error words and trace frames
__global__ void hbm_finish_kernel(DevProg P, RunArgs A, HbmState H, uint64_t batch0, uint32_t W) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  const uint64_t si0 = batch0 + (uint64_t)w * 32;
  const uint64_t nleft = A.nshots - si0;
  const uint32_t validmask = nleft >= 32 ? kFull : ((1u << nleft) - 1u);
  const uint32_t gw = (uint32_t)(si0 >> 5);
  for (int o = 0; o < P.O; o++) A.obs[(size_t)o * A.W + gw] = H.obs[(size_t)o * W + w] & validmask;
  A.accepted[gw] = H.alive[w] & validmask;
  A.error[gw] = H.err[w];
  for (int j = 0; j < 32; j++) {
    if (!((validmask >> j) & 1)) continue;
    const uint64_t si = si0 + j, bs = (uint64_t)w * 32 + j;
    if (A.t_fx && !((H.frozen[w] >> j) & 1))
      for (int q = 0; q < P.n; q++) {
        A.t_fx[si * P.n + q] = (H.fx[(size_t)q * W + w] >> j) & 1;
        A.t_fz[si * P.n + q] = (H.fz[(size_t)q * W + w] >> j) & 1;
      }
    if (A.t_gamma) { A.t_gamma[2 * si] = H.gamma[bs].x; A.t_gamma[2 * si + 1] = H.gamma[bs].y; }
    if (A.t_draws) A.t_draws[si] = H.smcount[bs];
  }
}

// trace checkpoint j: frames, gamma and validity of the shots still running (amplitudes: gather)
__global__ void hbm_cp_kernel(DevProg P, RunArgs A, HbmState H, uint64_t batch0, uint32_t W, int j) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  const uint64_t si0 = batch0 + (uint64_t)w * 32;
  const uint64_t nleft = A.nshots - si0;
  const uint32_t validmask = nleft >= 32 ? kFull : ((1u << nleft) - 1u);
  const uint32_t alive = H.alive[w] & validmask;
  for (int b = 0; b < 32; b++) {
    if (!((alive >> b) & 1)) continue;
    const uint64_t si = si0 + b, bs = (uint64_t)w * 32 + b;
    const size_t cs = (size_t)j * A.nshots + si;
    A.cp_valid[cs] = 1;
    for (int q = 0; q < P.n; q++) {
      A.cp_fx[cs * P.n + q] = (H.fx[(size_t)q * W + w] >> b) & 1;
      A.cp_fz[cs * P.n + q] = (H.fz[(size_t)q * W + w] >> b) & 1;
    }
    A.cp_gamma[2 * cs] = H.gamma[bs].x;
    A.cp_gamma[2 * cs + 1] = H.gamma[bs].y;
  }
}

// ------------------------------------------------------------------ array kernels
enum HbmArrOp : int {
  HA_INIT = 0, HA_S, HA_SDAG, HA_H, HA_CX, HA_CZ, HA_EXPAND, HA_ROT, HA_COLLAPSE, HA_ACTIVE_ZERO, HA_RETIRE, HA_GATHER
};

struct ArrOp {
  int kind;
  int pa, pb;        // physical axes
  int k;             // logical dimension the op works at (elements enumerated = 2^k / touched fraction)
  int instr;         // instruction index (parity words)
  double2 c0, c1;    // phases (rot / expand: parity-0 pair, c2/c3 for parity 1)
  double2 c2, c3;
  DeadBits dead;     // dead physical positions (ascending) for the current valid set
};

// enumerate `count` logical work items over (shot, item) and apply the op
__global__ void __launch_bounds__(256) hbm_array_kernel(ArrOp o, HbmState H, uint64_t count_per_shot, uint32_t W) {
  const uint32_t shot = blockIdx.y;
  const uint32_t w = shot >> 5;
  const uint32_t bit = 1u << (shot & 31);
  if (!(H.alive[w] & bit)) return;
  double2* __restrict__ A = H.amps + (size_t)shot * H.cap;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count_per_shot;
       j += (uint64_t)gridDim.x * blockDim.x) {
    switch (o.kind) {
      case HA_S:
      case HA_SDAG: {  // elements with bit pa set: logical item j over k-1 other axes
        uint64_t i = o.dead.expand(j) | (1ull << o.pa);
        double2 v = A[i];
        A[i] = o.kind == HA_S ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
        break;
      }
      case HA_H: {
        uint64_t i0 = o.dead.expand(j);
        uint64_t i1 = i0 | (1ull << o.pa);
        double2 lo = A[i0], hi = A[i1];
        A[i0] = cscale(cadd(lo, hi), kInvSqrt2);
        A[i1] = cscale(csub(lo, hi), kInvSqrt2);
        break;
      }
      case HA_CX: {
        uint64_t i = o.dead.expand(j) | (1ull << o.pa);
        uint64_t i1 = i | (1ull << o.pb);
        double2 t = A[i];
        A[i] = A[i1];
        A[i1] = t;
        break;
      }
      case HA_CZ: {
        uint64_t i = o.dead.expand(j) | (1ull << o.pa) | (1ull << o.pb);
        double2 v = A[i];
        A[i] = make_double2(-v.x, -v.y);
        break;
      }
      case HA_ROT: {
        const int par = (H.par[(size_t)o.instr * W + w] & bit) ? 1 : 0;
        const double2 e0 = o.c0, e1 = o.c1;
        const double2 ph0 = par ? e1 : e0, ph1 = par ? e0 : e1;
        uint64_t i0 = o.dead.expand(j);
        uint64_t i1 = i0 | (1ull << o.pa);
        A[i0] = cmul(A[i0], ph0);
        A[i1] = cmul(A[i1], ph1);
        break;
      }
      case HA_EXPAND: {  // pa = the (dead) physical axis that becomes live; dead set excludes pa
        const int par = (H.par[(size_t)o.instr * W + w] & bit) ? 1 : 0;
        const double2 ph0 = par ? o.c2 : o.c0, ph1 = par ? o.c3 : o.c1;
        uint64_t i0 = o.dead.expand(j);
        uint64_t i1 = i0 | (1ull << o.pa);
        double2 v = A[i0];
        A[i0] = cmul(v, ph0);
        A[i1] = cmul(v, ph1);
        break;
      }
      case HA_COLLAPSE: {
        const double2 k0 = H.kco[2 * (size_t)shot], k1 = H.kco[2 * (size_t)shot + 1];
        uint64_t i0 = o.dead.expand(j);
        uint64_t i1 = i0 | (1ull << o.pa);
        A[i0] = cadd(cmul(k0, A[i0]), cmul(k1, A[i1]));
        break;
      }
      case HA_ACTIVE_ZERO: {  // MeasActive: zero the dead half, scale the live half
        const int br = (H.brw[w] & bit) ? 1 : 0;
        const double s = H.kco[2 * (size_t)shot].x;
        const bool renorm = o.c0.x != 0.0;
        uint64_t i0 = o.dead.expand(j);
        uint64_t i1 = i0 | (1ull << o.pa);
        uint64_t idead = br ? i0 : i1, ilive = br ? i1 : i0;
        A[idead] = make_double2(0.0, 0.0);
        if (renorm) A[ilive] = cscale(A[ilive], s);
        break;
      }
      case HA_RETIRE: {  // move the surviving half into the bit-0 position
        const int br = (H.brw[w] & bit) ? 1 : 0;
        if (br) {
          uint64_t i0 = o.dead.expand(j);
          A[i0] = A[i0 | (1ull << o.pa)];
        }
        break;
      }
      default: break;
    }
  }
}

// per-shot partial sums for a measurement: p1 = sum |u10 a0 + u11 a1|^2 (or sum |a1|^2 for
// MeasActive), p_all = sum |a|^2; fixed-order two-level reduction (deterministic)
__global__ void __launch_bounds__(256) hbm_reduce_kernel(ArrOp o, HbmState H, uint64_t pairs, int collapse,
                                                         double2 u10, double2 u11) {
  const uint32_t shot = blockIdx.y;
  const uint32_t w = shot >> 5, bit = 1u << (shot & 31);
  double s1 = 0.0, sa = 0.0;
  if (H.alive[w] & bit) {
    const double2* __restrict__ A = H.amps + (size_t)shot * H.cap;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < pairs; j += (uint64_t)gridDim.x * blockDim.x) {
      uint64_t i0 = o.dead.expand(j);
      double2 a0 = A[i0], a1 = A[i0 | (1ull << o.pa)];
      if (collapse) s1 = __dadd_rn(s1, cnorm2(cadd(cmul(a0, u10), cmul(u11, a1))));
      else s1 = __dadd_rn(s1, cnorm2(a1));
      sa = __dadd_rn(sa, __dadd_rn(cnorm2(a0), cnorm2(a1)));
    }
  }
  __shared__ double r1[256], ra[256];
  r1[threadIdx.x] = s1;
  ra[threadIdx.x] = sa;
  __syncthreads();
  for (int st = 128; st; st >>= 1) {
    if (threadIdx.x < st) {
      r1[threadIdx.x] = __dadd_rn(r1[threadIdx.x], r1[threadIdx.x + st]);
      ra[threadIdx.x] = __dadd_rn(ra[threadIdx.x], ra[threadIdx.x + st]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    H.red[((size_t)shot * H.nblk + blockIdx.x) * 2] = r1[0];
    H.red[((size_t)shot * H.nblk + blockIdx.x) * 2 + 1] = ra[0];
  }
}

__global__ void hbm_reduce_final_kernel(HbmState H, uint32_t nshots_batch, int nblk_used) {
  const uint32_t shot = blockIdx.x * blockDim.x + threadIdx.x;
  if (shot >= nshots_batch) return;
  double s1 = 0.0, sa = 0.0;
  for (int b = 0; b < nblk_used; b++) {
    s1 = __dadd_rn(s1, H.red[((size_t)shot * H.nblk + b) * 2]);
    sa = __dadd_rn(sa, H.red[((size_t)shot * H.nblk + b) * 2 + 1]);
  }
  H.p1[shot] = s1;
  H.pall[shot] = sa;
}

// initialise amplitude 0 of every shot (the rest is written before being read)
__global__ void hbm_init_amps_kernel(HbmState H, uint32_t nshots_batch) {
  const uint32_t shot = blockIdx.x * blockDim.x + threadIdx.x;
  if (shot < nshots_batch) H.amps[(size_t)shot * H.cap] = make_double2(1.0, 0.0);
}

// trace: gather the valid elements of each shot in logical order into dst [nshots][2^k][2]
__global__ void hbm_gather_kernel(DevProg P, RunArgs A, HbmState H, uint64_t batch0, uint32_t nshots_batch,
                                  int k, DevAxisMap map, double* dst) {
  const uint32_t shot = blockIdx.y;
  if (shot >= nshots_batch) return;
  const uint64_t sz = 1ull << k;
  const uint64_t si = batch0 + shot;
  const double2* A_ = H.amps + (size_t)shot * H.cap;
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < sz; l += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t p = 0;
    for (int b = 0; b < k; b++) p |= ((l >> b) & 1ull) << map.phys[b];
    const double2 v = A_[p];
    dst[(si * sz + l) * 2] = v.x;
    dst[(si * sz + l) * 2 + 1] = v.y;
  }
}

}  // namespace fs
