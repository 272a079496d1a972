// fs_frame.cuh -- the bit-sliced frame engine for frame-only programs (k_max = 0, e.g. the
// surface-code memory of config 1).
//
// Each LANE owns one 32-shot word, so a warp advances 1024 shots per instruction with no
// cross-lane communication at all.  The Pauli frame is bit-sliced across shots: smem words
// fx[q][lane], fz[q][lane] (bank = lane, conflict-free).  Frame gates become word XORs/swaps,
// records are words written straight to the [record][word] output (a warp stores 128 B per
// record, fully coalesced), detectors/observables are word XORs of slot words, random
// dormant measurements use one Philox word (32 coins) per word, and noise uses the
// word-level flattened hazard process (one Exp(1) jump per realised fault over 32 lanes).
#pragma once
#include "fs_general.cuh"

namespace fs {

constexpr int kFrameWarps = 4;

__device__ __forceinline__ void word_gate_strided(uint32_t* fx, uint32_t* fz, uint32_t g) {
  const int a = FS_GATE_A(g) * 32, b = FS_GATE_B(g) * 32;
  uint32_t t;
  switch (FS_GATE_G(g)) {
    case FS_G_H: t = fx[a]; fx[a] = fz[a]; fz[a] = t; break;
    case FS_G_S:
    case FS_G_SDAG: fz[a] ^= fx[a]; break;
    case FS_G_CX: fx[b] ^= fx[a]; fz[a] ^= fz[b]; break;
    case FS_G_CZ: fz[b] ^= fx[a]; fz[a] ^= fx[b]; break;
    case FS_G_SWAP:
      t = fx[a]; fx[a] = fx[b]; fx[b] = t;
      t = fz[a]; fz[a] = fz[b]; fz[b] = t;
      break;
    default: break;
  }
}

struct PhiloxDraw {  // per-shot Philox stream used by forced fault modes 0/1
  PhiloxStream ps;
  __device__ __forceinline__ double uniform() { return ps.uniform(); }
};

template <bool TRACE>
__global__ void __launch_bounds__(kFrameWarps * 32)
frame_kernel(DevProg P, RunArgs A, int smem_words_per_warp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* base = reinterpret_cast<uint32_t*>(smem_raw) + (size_t)wib * smem_words_per_warp * 32 + lane;
  uint32_t* fx = base;
  uint32_t* fz = base + P.n * 32;
  uint32_t* slots = fz + P.n * 32;
  uint32_t* obsw = slots + P.num_slots * 32;
  const uint64_t word0 = A.shot0 >> 5;
  const int nwords_smem = 2 * P.n + P.num_slots + P.O;

  for (uint32_t w = (blockIdx.x * kFrameWarps + wib) * 32 + lane; w < A.W; w += gridDim.x * kFrameWarps * 32) {
    const uint64_t wabs = word0 + w;
    const uint64_t nleft = A.nshots - (uint64_t)w * 32;
    const uint32_t validmask = nleft >= 32 ? kFull : ((1u << nleft) - 1u);
    uint32_t alive = validmask, errmask = 0;
    int errcode = 0;
    for (int q = 0; q < nwords_smem; q++) base[q * 32] = 0;
    FaultBuffer<kFaultCap> fbuf;
    if (!(TRACE && A.fault_modes)) fbuf.init(P, A.seed, wabs);
    uint32_t dumped = 0;
    auto dump_frames = [&](uint32_t mask) {
      for (int j = 0; j < 32; j++) {
        if (!((mask >> j) & 1)) continue;
        const uint64_t si = (uint64_t)w * 32 + j;
        for (int q = 0; q < P.n; q++) {
          A.t_fx[si * P.n + q] = (fx[q * 32] >> j) & 1;
          A.t_fz[si * P.n + q] = (fz[q * 32] >> j) & 1;
        }
      }
    };

    for (int i = 0; i < A.stop; i++) {
      const int4 I0 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i);
      const int4 I1 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i + 1);
      const int op = FS_OPCODE(I0.x);
      const uint32_t flipw = FS_FLIP(I0.x) ? kFull : 0u;
      switch (op) {
        case FS_OP_FRAME: {
          const int off = I0.y, cnt = I0.z;
          for (int j = 0; j < cnt; j++) word_gate_strided(fx, fz, __ldg(P.gates + off + j));
          break;
        }
        case FS_OP_MEAS_DSTATIC:
        case FS_OP_MEAS_DRANDOM: {
          const int virt = I0.y, rec = I0.w;
          uint32_t recw;
          if (op == FS_OP_MEAS_DSTATIC) {
            recw = fx[virt * 32] ^ flipw;
            if (TRACE && A.forced) {
              uint32_t bad = 0;
              for (int j = 0; j < 32; j++) {
                if (!((alive >> j) & 1)) continue;
                int fo = A.forced[((uint64_t)w * 32 + j) * P.R + rec];
                if (fo >= 0 && fo != (int)((recw >> j) & 1)) bad |= 1u << j;
              }
              if (bad) { errmask |= bad; alive &= ~bad; errcode = FS_ERR_SHOT_FORCED; }
            }
          } else {
            const uint32_t pw = fz[virt * 32];
            uint32_t coinw = coin_word(A.seed, wabs, I0.z);
            if (TRACE && A.forced) {
              for (int j = 0; j < 32; j++) {
                if (!((validmask >> j) & 1)) continue;
                int fo = A.forced[((uint64_t)w * 32 + j) * P.R + rec];
                if (fo >= 0) {
                  uint32_t c = (uint32_t)(fo ^ (int)((pw >> j) & 1) ^ (int)(flipw & 1));
                  coinw = (coinw & ~(1u << j)) | (c << j);
                }
              }
            }
            const uint32_t t = fx[virt * 32];
            fx[virt * 32] = fz[virt * 32] ^ coinw;
            fz[virt * 32] = t;
            recw = coinw ^ pw ^ flipw;
          }
          const int col = __ldg(P.record_out + rec);
          if (col >= 0) A.meas[(size_t)col * A.W + w] = recw & alive;
          const int sl = __ldg(P.bit_slot + rec);
          if (sl >= 0) slots[sl * 32] = recw;
          break;
        }
        case FS_OP_COND_FRAME: {
          const uint32_t rw = slots[__ldg(P.bit_slot + I0.w) * 32];
          if (rw) {
            for (int j = 0; j < I0.z; j++) {
              uint32_t e = __ldg(P.paulis + I0.y + j);
              (FS_PAULI_Z(e) ? fz : fx)[FS_PAULI_Q(e) * 32] ^= rw;
            }
          }
          break;
        }
        case FS_OP_NOISE: {
          const int ins[8] = {I0.x, I0.y, I0.z, I0.w, I1.x, I1.y, I1.z, I1.w};
          if (TRACE && A.fault_modes) {
            for (int j = 0; j < 32; j++) {
              if (!((alive >> j) & 1)) continue;
              const uint64_t si = (uint64_t)w * 32 + j;
              PhiloxDraw d;
              d.ps.init(A.seed, A.shot0 + si, (uint32_t)i, TAG_FORCED);
              forced_faults_shot(P, fx, fz, 1u << j, ins, A.fault_modes + si * P.E, d, 32);
            }
          } else {
            fbuf.apply_until(P, I0.z, [&](int c, int l) {
              const int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
              for (int j = off; j < end; j++) {
                const uint32_t e = __ldg(P.paulis + j);
                (FS_PAULI_Z(e) ? fz : fx)[FS_PAULI_Q(e) * 32] ^= 1u << l;
              }
            });
          }
          break;
        }
        case FS_OP_DETECTOR:
        case FS_OP_OBSERVABLE: {
          uint32_t wv = 0;
          for (int j = 0; j < I0.w; j++) wv ^= slots[__ldg(P.bit_slot + __ldg(P.reclists + I0.z + j)) * 32];
          if (op == FS_OP_DETECTOR) {
            A.det[(size_t)I0.y * A.W + w] = wv & alive;
            const int sl = __ldg(P.bit_slot + P.R + I0.y);
            if (sl >= 0) slots[sl * 32] = wv;
          } else {
            obsw[I0.y * 32] ^= wv & alive;
          }
          break;
        }
        case FS_OP_POSTSELECT: {
          const int bid = I0.y == 0 ? P.R + I0.z : I0.z;
          const uint32_t bw = slots[__ldg(P.bit_slot + bid) * 32];
          const uint32_t rej = (bw ^ (I0.w ? kFull : 0u)) & alive;
          alive &= ~rej;
          if (TRACE && rej && A.t_fx) {  // a rejected shot's frame freezes at its halt point
            dump_frames(rej);
            dumped |= rej;
          }
          break;
        }
        default: break;  // GammaRot: global phase only, no observable effect
      }
    }
    for (int o = 0; o < P.O; o++) A.obs[(size_t)o * A.W + w] = obsw[o * 32] & validmask;
    A.accepted[w] = alive & validmask;
    A.error[w] = errmask;
    if (errmask) atomicMax(A.status, errcode);
    if (TRACE && A.t_fx) dump_frames(validmask & ~dumped);
  }
}

}  // namespace fs
