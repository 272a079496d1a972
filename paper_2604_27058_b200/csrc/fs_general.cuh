// fs_general.cuh -- the general engine: one warp executes one 32-shot word, lane = shot.
//
// Every opcode of the reference VM (runtime.py:130-641) is implemented.  State per warp:
//   * Pauli frame bit-sliced across the warp's 32 shots: smem word fx[q], fz[q] (bit = lane);
//     word-level updates are issued by lane 0 and published with __syncwarp;
//   * record / detector bits that a later instruction reads: smem slot words (program.py slot
//     allocation), every other record goes straight to the output words;
//   * per-lane dense active array of 2^k complex128, interleaved [i][lane] so a warp-wide
//     access is one coalesced 512 B row, in shared memory when 32*2^k_max*16 B fits, else in a
//     per-resident-warp HBM scratch slab;
//   * per-lane gamma, random stream and trace inputs.
#pragma once
#include "fs_device.cuh"

namespace fs {

constexpr int kGenWarps = 4;  // warps per block of the general engine

__device__ __forceinline__ void word_gate(uint32_t* fx, uint32_t* fz, uint32_t g) {
  int a = FS_GATE_A(g), b = FS_GATE_B(g);
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

// XOR the Pauli list [off, off+cnt) into frame words with `bits` (lane-0 writer or atomics)
template <bool ATOMIC>
__device__ __forceinline__ void xor_paulis(const DevProg& P, uint32_t* fx, uint32_t* fz, int off, int cnt,
                                           uint32_t bits) {
  for (int j = 0; j < cnt; j++) {
    uint32_t e = __ldg(P.paulis + off + j);
    uint32_t* f = FS_PAULI_Z(e) ? fz : fx;
    if (ATOMIC) atomicXor(f + FS_PAULI_Q(e), bits);
    else f[FS_PAULI_Q(e)] ^= bits;
  }
}

__device__ __forceinline__ void xor_case(const DevProg& P, uint32_t* fx, uint32_t* fz, int c, uint32_t bits,
                                         bool atomic) {
  int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
  if (atomic) xor_paulis<true>(P, fx, fz, off, end - off, bits);
  else xor_paulis<false>(P, fx, fz, off, end - off, bits);
}

// Philox noise stream: one geometric-skip process per 32-shot word over the
// whole program (runs of equal-probability sites, site-major (site, lane) cells), generated
// lazily into a small per-thread buffer and consumed in site order by the NoiseBlocks.
struct WordFaultGen {
  uint64_t seed, wabs;
  uint32_t step_no;
  int run;
  int cl;    // next lane of a certain site
  double c;  // current cell of a geometric run
  __device__ __forceinline__ void init(uint64_t s, uint64_t w) {
    seed = s;
    wabs = w;
    step_no = 0;
    run = 0;
    cl = 0;
    c = -1.0;
  }
  // One step = one Philox block: 0 nothing emitted, 1 fault (site, lane, case), 2 exhausted.
  __device__ __forceinline__ int step(const DevProg& P, int& site, int& lane, int& cs) {
    if (run >= P.num_runs) return 2;
    const int start = __ldg(P.run_start + run), len = __ldg(P.run_len + run);
    const uint4 b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), 0u, (TAG_NOISE << 24) | step_no++, seed);
    const double u2 = u64_to_unit(((uint64_t)b.w << 32) | b.z);
    if (len == 0) {  // certain site: lane cl fires
      site = start;
      lane = cl++;
      if (cl == 32) { run++; cl = 0; }
      cs = __ldg(P.site_case_off + site);
      if (num_cases(P, site) > 1) cs = pick_case(P, site, u2);
      return 1;
    }
    const double g = floor(__dmul_rn(ln_unit(((uint64_t)b.y << 32) | b.x), __ldg(P.run_lp + run)));
    c = __dadd_rn(__dadd_rn(c, 1.0), g);
    if (!(c < (double)(32 * len))) { run++; c = -1.0; return 0; }
    const long long ci = (long long)c;
    lane = (int)(ci & 31);
    site = start + (int)(ci >> 5);
    const double x = __dmul_rn(u2, __ldg(P.run_q + run));  // uniform on [0, q)
    if (!(x < __ldg(P.site_prob + site))) return 0;        // thinning: p_site < q
    cs = __ldg(P.site_case_off + site);
    if (num_cases(P, site) > 1) cs = pick_case_x(P, site, x);
    return 1;
  }
  // step() in two halves for a consumer that owns one lane of the word: first the candidate --
  // (site, lane), its uniform, whether the site is a certain one -- from the same Philox block and
  // with the same stream position as step(); the thinning test and the case pick (dependent table
  // loads, most of a step's latency) only for the candidates the consumer keeps (resolve)
  __device__ __forceinline__ int step_cand(const DevProg& P, int& site, int& lane, double& x, int& certain) {
    if (run >= P.num_runs) return 2;
    const uint4 b = philox((uint32_t)wabs, (uint32_t)(wabs >> 32), 0u, (TAG_NOISE << 24) | step_no, seed);
    return step_with(P, ln_unit(((uint64_t)b.y << 32) | b.x), u64_to_unit(((uint64_t)b.w << 32) | b.z), site, lane, x, certain);
  }
  // the stream-position half of step_cand, given the step's two draws (L = ln of the gap uniform,
  // u2 = the thinning / case uniform): consumers that draw a batch of steps at once (fs_wseg.cuh)
  __device__ __forceinline__ int step_with(const DevProg& P, double L, double u2, int& site, int& lane, double& x,
                                           int& certain) {
    const int start = __ldg(P.run_start + run), len = __ldg(P.run_len + run);
    step_no++;
    if (len == 0) {
      site = start;
      lane = cl++;
      if (cl == 32) { run++; cl = 0; }
      x = u2;
      certain = 1;
      return 1;
    }
    const double g = floor(__dmul_rn(L, __ldg(P.run_lp + run)));
    c = __dadd_rn(__dadd_rn(c, 1.0), g);
    if (!(c < (double)(32 * len))) { run++; c = -1.0; return 0; }
    const long long ci = (long long)c;
    lane = (int)(ci & 31);
    site = start + (int)(ci >> 5);
    x = __dmul_rn(u2, __ldg(P.run_q + run));  // uniform on [0, q)
    certain = 0;
    return 1;
  }
  // the case of a candidate, or -1 when thinning drops it
  __device__ __forceinline__ static int resolve(const DevProg& P, int site, double x, int certain) {
    if (!certain && !(x < __ldg(P.site_prob + site))) return -1;
    int cs = __ldg(P.site_case_off + site);
    if (num_cases(P, site) > 1) cs = certain ? pick_case(P, site, x) : pick_case_x(P, site, x);
    return cs;
  }
};

template <int CAP>
struct FaultBuffer {
  WordFaultGen gen;
  int cnt, cur;
  bool more;
  int fsite[CAP];
  uint32_t fent[CAP];  // absolute case << 5 | lane
  __device__ __forceinline__ void refill(const DevProg& P) {
    cnt = 0;
    cur = 0;
    int site = 0, lane = 0, cs = 0;
    for (;;) {  // one Philox block per iteration: keeps the lanes of a warp in lock step
      const int r = gen.step(P, site, lane, cs);
      if (r == 2) { more = false; return; }
      if (r == 1) {
        fsite[cnt] = site;
        fent[cnt] = ((uint32_t)cs << 5) | (uint32_t)lane;
        if (++cnt == CAP) return;
      }
    }
  }
  __device__ __forceinline__ void init(const DevProg& P, uint64_t seed, uint64_t wabs) {
    gen.init(seed, wabs);
    more = true;
    refill(P);
  }
  // apply (via fn(case, lane)) every buffered fault with site < hi
  template <class Fn>
  __device__ __forceinline__ void apply_until(const DevProg& P, int hi, Fn&& fn) {
    for (;;) {
      if (cur == cnt) {
        if (!more) return;
        refill(P);
        if (cnt == 0) return;
      }
      if (fsite[cur] >= hi) return;
      const uint32_t e = fent[cur++];
      fn((int)(e >> 5), (int)(e & 31));
    }
  }
};

constexpr int kFaultCap = 48;

// Reference hazard skipping for one shot (runtime.py:564-586 / :675-699), draw for draw.
// Frame words are `stride` apart; `atomic` when several lanes share the words.
__device__ __forceinline__ void xor_case_strided(const DevProg& P, uint32_t* fx, uint32_t* fz, int c, uint32_t bit,
                                                 int stride, bool atomic) {
  int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
  for (int j = off; j < end; j++) {
    uint32_t e = __ldg(P.paulis + j);
    uint32_t* f = (FS_PAULI_Z(e) ? fz : fx) + (size_t)FS_PAULI_Q(e) * stride;
    if (atomic) atomicXor(f, bit);
    else *f ^= bit;
  }
}

template <class Draw>
__device__ void hazard_shot(const DevProg& P, uint32_t* fx, uint32_t* fz, uint32_t bit, const int* ins, Draw& rng,
                            int stride = 1, bool atomic = true) {
  const double* S = P.cum_hazard;
  const int plan_off = ins[3], plan_cnt = ins[4];
  for (int pi = 0; pi < plan_cnt; pi++) {
    int a = __ldg(P.plans + 2 * (plan_off + pi)), b = __ldg(P.plans + 2 * (plan_off + pi) + 1);
    if (a < 0) {
      int site = b, c = __ldg(P.site_case_off + site);
      if (num_cases(P, site) > 1) c = pick_case(P, site, rng.uniform());
      xor_case_strided(P, fx, fz, c, bit, stride, atomic);
      continue;
    }
    int i = a;
    while (i < b) {
      double target = __dadd_rn(__ldg(S + i), -log1p(-rng.uniform()));
      int idx = bisect_right(S, target, i + 1, b + 1);
      if (idx > b) break;
      int site = idx - 1, c = __ldg(P.site_case_off + site);
      if (num_cases(P, site) > 1) c = pick_case(P, site, rng.uniform());
      xor_case_strided(P, fx, fz, c, bit, stride, atomic);
      i = site + 1;
    }
  }
}

// Forced fault modes for one shot (runtime.py:587-601).  stride==1 => words shared by lanes (atomic).
template <class Draw>
__device__ void forced_faults_shot(const DevProg& P, uint32_t* fx, uint32_t* fz, uint32_t bit, const int* ins,
                                   const int16_t* modes, Draw& rng, int stride, bool atomic = false) {
  for (int site = ins[1]; site < ins[2]; site++) {
    int mode = modes[site];
    if (mode == 2) continue;
    int nc = num_cases(P, site);
    int c = __ldg(P.site_case_off + site);
    if (mode == 0) {
      if (nc == 0) continue;
      if (rng.uniform() >= __ldg(P.site_prob + site)) continue;
      if (nc > 1) c = pick_case(P, site, rng.uniform());
    } else if (mode == 1) {
      if (nc > 1) c = pick_case(P, site, rng.uniform());
    } else {
      c += mode - 3;
    }
    xor_case_strided(P, fx, fz, c, bit, stride, atomic);
  }
}

// per-shot draw source for the general engine: SplitMix (reference) or Philox (per shot/instr)
struct ShotDraws {
  bool splitmix;
  SplitMix sm;
  PhiloxStream ph;
  uint64_t seed, shot;
  __device__ __forceinline__ void begin(int instr, uint32_t tag) {
    if (!splitmix) ph.init(seed, shot, (uint32_t)instr, tag);
  }
  __device__ __forceinline__ double uniform() { return splitmix ? sm.uniform() : ph.uniform(); }
};

// Segmented mode (programs with PostSelect): the program is cut after every PostSelect; each
// segment runs over the list of shots still alive, 32 per warp (lanes carry arbitrary shot
// ids), and the survivors' state is compacted into a store for the next segment.
struct StateStore {
  uint32_t* frame;    // [slot][nfw]  packed x bits (q) then z bits (n+q)
  uint32_t* slotbits; // [slot][nsw]
  uint32_t* obsbits;  // [slot][now]
  double2* gamma;     // [slot]
  uint32_t* smcount;  // [slot]
  uint32_t* gen_i;    // [slot][6]: step_no, run, cl, pend_site, pend_lane, pend_case
  double* gen_c;      // [slot]
  double2* amps;      // [slot/32][cap][32] (interleaved) or [slot][cap] (shot_major)
  uint32_t* shot;     // [slot] shot index within the call
  int shot_major;     // layout chosen for the consuming engine
};

// amplitude j of store slot `slot`: interleaved [slot/32][j][32] or shot-major [slot][j]
__device__ __forceinline__ size_t store_amp_index(uint32_t slot, uint32_t j, uint32_t cap, int shot_major) {
  return shot_major ? (size_t)slot * cap + j : (size_t)(slot >> 5) * ((size_t)cap * 32) + (size_t)j * 32 + (slot & 31);
}

struct SegArgs {
  int seg_begin, seg_end;  // instruction range of this segment
  int first, last;         // initialise / finalise
  uint32_t n_in;
  uint64_t chunk0;         // first shot (within the call) of the chunk (identity list)
  uint32_t* n_out;         // survivors counter
  StateStore in, out;
  int k_in, k_out;         // active dimension at the segment boundaries
  int nfw, nsw, now;
  int fuse;                // block engine: star groups enabled (no checkpoint falls inside one)
};

template <bool SPLITMIX, bool ARR_SMEM, bool SEG>
__global__ void __launch_bounds__(kGenWarps * 32)
general_kernel(DevProg P, RunArgs A, int smem_words_per_warp, SegArgs S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t lanebit = 1u << lane;
  uint32_t* wsm = reinterpret_cast<uint32_t*>(smem_raw) + (size_t)wib * smem_words_per_warp;
  uint32_t* fx = wsm;
  uint32_t* fz = fx + P.n;
  uint32_t* slots = fz + P.n;
  uint32_t* obsw = slots + P.num_slots;
  const size_t cap = (size_t)1 << A.arr_log2;
  double2* arr;
  if (ARR_SMEM) {
    unsigned char* abase = smem_raw + (size_t)kGenWarps * smem_words_per_warp * 4;
    abase = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(abase) + 15) & ~uintptr_t(15));
    arr = reinterpret_cast<double2*>(abase) + (size_t)wib * cap * 32;
  } else {
    const size_t gwarp = (size_t)blockIdx.x * kGenWarps + wib;
    arr = A.scratch + gwarp * cap * 32;
  }
#define AMP(i) arr[(size_t)(i) * 32 + lane]
  const bool renorm = !(A.flags & FS_NO_RENORM);
  const uint64_t word0 = A.shot0 >> 5;
  const int stop = A.stop;
  const int i_begin = SEG ? S.seg_begin : 0;
  const int i_end = SEG ? S.seg_end : stop;
  const uint32_t nunits = SEG ? (S.n_in + 31) / 32 : A.W;

  for (uint32_t w = blockIdx.x * kGenWarps + wib; w < nunits; w += gridDim.x * kGenWarps) {
    const uint32_t idx = w * 32 + lane;  // SEG: input slot of this lane
    uint64_t si;                          // shot index within the call
    bool valid;
    if (SEG) {
      valid = idx < S.n_in;
      si = S.first ? S.chunk0 + idx : (valid ? S.in.shot[idx] : 0);
      valid = valid && si < A.nshots;
    } else {
      si = (uint64_t)w * 32 + lane;
      valid = si < A.nshots;
    }
    const uint64_t shot = A.shot0 + si;
    const uint64_t wabs = SEG ? (shot >> 5) : word0 + w;  // SEG: the lane's own 32-shot word
    const uint32_t wout = SEG ? (uint32_t)((S.chunk0 >> 5) + w) : w;  // output word (aligned)
    const bool aligned = !SEG || S.first;  // lanes == consecutive shots of one output word
    const uint32_t validmask = __ballot_sync(kFull, valid);
    uint32_t alive = validmask;
    uint32_t errmask = 0;
    int errcode = 0;
    for (int q = lane; q < 2 * P.n + P.num_slots + P.O; q += 32) wsm[q] = 0;
    AMP(0) = make_double2(1.0, 0.0);
    double2 gamma = make_double2(1.0, 0.0);
    ShotDraws rng;
    rng.splitmix = SPLITMIX;
    rng.seed = A.seed;
    rng.shot = shot;
    if (SPLITMIX) rng.sm.reset(A.seed, shot);
    if (SPLITMIX && A.draw0 && valid) rng.sm.count = A.draw0[si];
    const int16_t* fmodes = A.fault_modes ? A.fault_modes + (valid ? si : 0) * (size_t)P.E : nullptr;
    const int8_t* forced = A.forced ? A.forced + (valid ? si : 0) * (size_t)P.R : nullptr;
    int branch = 0;
    FaultBuffer<kFaultCap> fbuf;
    if (!SEG && !SPLITMIX && !fmodes && lane == 0) fbuf.init(P, A.seed, wabs);
    // SEG + Philox: every lane runs its own word's generator lazily, keeping one pending fault
    WordFaultGen lgen;
    int pend_site = -1, pend_lane = 0, pend_case = 0;
    if (SEG && !SPLITMIX) lgen.init(A.seed, wabs);
    __syncwarp();
    if (SEG && !S.first) {  // restore the survivor state saved by the previous segment
      const StateStore& I = S.in;
      for (int b = 0; b < 2 * P.n; b++) {
        const int bit = valid ? (int)((I.frame[(size_t)idx * S.nfw + (b >> 5)] >> (b & 31)) & 1) : 0;
        const uint32_t wv = __ballot_sync(kFull, bit);
        if (lane == 0) { if (b < P.n) fx[b] = wv; else fz[b - P.n] = wv; }
      }
      for (int b = 0; b < P.num_slots; b++) {
        const int bit = valid ? (int)((I.slotbits[(size_t)idx * S.nsw + (b >> 5)] >> (b & 31)) & 1) : 0;
        const uint32_t wv = __ballot_sync(kFull, bit);
        if (lane == 0) slots[b] = wv;
      }
      for (int b = 0; b < P.O; b++) {
        const int bit = valid ? (int)((I.obsbits[(size_t)idx * S.now + (b >> 5)] >> (b & 31)) & 1) : 0;
        const uint32_t wv = __ballot_sync(kFull, bit);
        if (lane == 0) obsw[b] = wv;
      }
      if (valid) {
        gamma = I.gamma[idx];
        if (SPLITMIX) rng.sm.count = I.smcount[idx];
        else {
          lgen.step_no = I.gen_i[(size_t)idx * 6];
          lgen.run = (int)I.gen_i[(size_t)idx * 6 + 1];
          lgen.cl = (int)I.gen_i[(size_t)idx * 6 + 2];
          pend_site = (int)I.gen_i[(size_t)idx * 6 + 3];
          pend_lane = (int)I.gen_i[(size_t)idx * 6 + 4];
          pend_case = (int)I.gen_i[(size_t)idx * 6 + 5];
          lgen.c = I.gen_c[idx];
        }
        const uint32_t sz = 1u << S.k_in;
        for (uint32_t j = 0; j < sz; j++) AMP(j) = I.amps[store_amp_index(idx, j, sz, I.shot_major)];
      }
      __syncwarp();
    }

    // write one record word to its output column and/or slot
    // one output bit row: whole word when the lanes are one output word, else per-lane bits
    auto put_out = [&](uint32_t* row, uint32_t word) {
      if (aligned) {
        if (lane == 0) row[wout] = word & alive;
      } else if (((word & alive) >> lane) & 1) {
        atomicOr(row + (si >> 5), 1u << (si & 31));
      }
    };
    auto put_record = [&](int r, uint32_t word) {
      if (A.t_rec && ((alive >> lane) & 1)) A.t_rec[si * P.R + r] = (uint8_t)((word >> lane) & 1);
      const int col = __ldg(P.record_out + r);
      if (col >= 0) put_out(A.meas + (size_t)col * A.W, word);
      if (lane == 0) {
        const int sl = __ldg(P.bit_slot + r);
        if (sl >= 0) slots[sl] = word;
      }
    };
    auto fail = [&](bool bad, int code) {
      uint32_t b = __ballot_sync(kFull, bad);
      if (b) {
        errmask |= b;
        alive &= ~b;
        errcode = code;
      }
    };

    // trace state of shots in `mask` as of now (a post-selected shot freezes at its halt point,
    // runtime.py:632-641, while the warp keeps executing for the others)
    uint32_t dumped = 0;
    auto dump_trace = [&](uint32_t mask, int upto) {
      if (!((mask >> lane) & 1)) return;
      if (A.t_fx)
        for (int q = 0; q < P.n; q++) {
          A.t_fx[si * P.n + q] = (fx[q] >> lane) & 1;
          A.t_fz[si * P.n + q] = (fz[q] >> lane) & 1;
        }
      if (A.t_gamma) { A.t_gamma[2 * si] = gamma.x; A.t_gamma[2 * si + 1] = gamma.y; }
      if (A.t_draws) A.t_draws[si] = SPLITMIX ? rng.sm.count : 0u;
      if (A.t_amps) {
        const int kst = stop > 0 ? __ldg(P.schedule + stop - 1) : 0;
        const int kcur = upto > 0 ? __ldg(P.schedule + upto - 1) : 0;
        const uint32_t sz = 1u << kst, cur = 1u << kcur;
        for (uint32_t j = 0; j < sz; j++) {
          double2 v = j < cur ? AMP(j) : make_double2(0.0, 0.0);
          A.t_amps[(si * sz + j) * 2] = v.x;
          A.t_amps[(si * sz + j) * 2 + 1] = v.y;
        }
      }
    };

    // checkpoint j: state after instructions [0, cp_at[j]) of the shots still running (a value
    // equal to a segment start was dumped at the end of the previous segment)
    auto dump_cp = [&](int j) {
      if (!((alive >> lane) & 1)) return;
      const size_t cs = (size_t)j * A.nshots + si;
      A.cp_valid[cs] = 1;
      for (int q = 0; q < P.n; q++) {
        A.cp_fx[cs * P.n + q] = (fx[q] >> lane) & 1;
        A.cp_fz[cs * P.n + q] = (fz[q] >> lane) & 1;
      }
      A.cp_gamma[2 * cs] = gamma.x;
      A.cp_gamma[2 * cs + 1] = gamma.y;
      const int c = __ldg(A.cp_at + j);
      const uint32_t sz = 1u << (c > 0 ? __ldg(P.schedule + c - 1) : 0);
      double* dst = A.cp_amps + 2 * (__ldg(A.cp_off + j) + si * sz);
      for (uint32_t e = 0; e < sz; e++) {
        const double2 v = AMP(e);
        dst[2 * e] = v.x;
        dst[2 * e + 1] = v.y;
      }
    };
    int cpi = 0;
    if (A.ncp) {
      const int lo = i_begin == 0 ? 0 : i_begin + 1;
      while (cpi < A.ncp && __ldg(A.cp_at + cpi) < lo) cpi++;
    }

    for (int i = i_begin; i < i_end; i++) {
      if (alive == 0 && A.prezeroed) break;
      while (cpi < A.ncp && __ldg(A.cp_at + cpi) == i) dump_cp(cpi++);
      const int4 I0 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i);
      const int4 I1 = __ldg(reinterpret_cast<const int4*>(P.instrs) + 2 * i + 1);
      const int ins[8] = {I0.x, I0.y, I0.z, I0.w, I1.x, I1.y, I1.z, I1.w};
      const int op = FS_OPCODE(I0.x);
      const uint32_t flipw = FS_FLIP(I0.x) ? kFull : 0u;
      const bool me = (alive >> lane) & 1;
      switch (op) {
        case FS_OP_FRAME: {
          if (lane == 0)
            for (int j = 0; j < ins[2]; j++) word_gate(fx, fz, __ldg(P.gates + ins[1] + j));
          __syncwarp();
          break;
        }
        case FS_OP_ARRAY_GATE: {
          const int g = ins[1], va = ins[2], vb = ins[3], a = ins[4], b = ins[5];
          const uint32_t size = 1u << ins[6];
          if (lane == 0) {
            uint32_t t;
            switch (g) {
              case FS_G_S: case FS_G_SDAG: fz[va] ^= fx[va]; break;
              case FS_G_H: t = fx[va]; fx[va] = fz[va]; fz[va] = t; break;
              case FS_G_CX: fx[vb] ^= fx[va]; fz[va] ^= fz[vb]; break;
              case FS_G_CZ: fz[vb] ^= fx[va]; fz[va] ^= fx[vb]; break;
            }
          }
          if (me) {
            if (g == FS_G_S || g == FS_G_SDAG) {
              const double2 ph = make_double2(0.0, g == FS_G_S ? 1.0 : -1.0);
              for (uint32_t j = 0; j < size / 2; j++) {
                uint32_t idx = ins0(j, a) | (1u << a);
                AMP(idx) = cmul(AMP(idx), ph);
              }
            } else if (g == FS_G_H) {
              const uint32_t st = 1u << a;
              for (uint32_t j = 0; j < size / 2; j++) {
                uint32_t i0 = ins0(j, a);
                double2 lo = AMP(i0), hi = AMP(i0 + st);
                AMP(i0) = cscale(cadd(lo, hi), kInvSqrt2);
                AMP(i0 + st) = cscale(csub(lo, hi), kInvSqrt2);
              }
            } else if (g == FS_G_CX) {
              const int lo_ax = a < b ? a : b, hi_ax = a < b ? b : a;
              for (uint32_t j = 0; j < size / 4; j++) {
                uint32_t idx = ins0(ins0(j, lo_ax), hi_ax) | (1u << a);
                uint32_t jdx = idx | (1u << b);
                double2 t0 = AMP(idx);
                AMP(idx) = AMP(jdx);
                AMP(jdx) = t0;
              }
            } else if (g == FS_G_CZ) {
              const int lo_ax = a < b ? a : b, hi_ax = a < b ? b : a;
              for (uint32_t j = 0; j < size / 4; j++) {
                uint32_t idx = ins0(ins0(j, lo_ax), hi_ax) | (1u << a) | (1u << b);
                double2 v = AMP(idx);
                AMP(idx) = make_double2(-v.x, -v.y);
              }
            }
          }
          __syncwarp();
          break;
        }
        case FS_OP_EXPAND: {
          const int par = (fx[ins[1]] >> lane) & 1;
          const double* f = P.fparams + ins[5] + 4 * par;
          const double2 ph0 = make_double2(__ldg(f), __ldg(f + 1)), ph1 = make_double2(__ldg(f + 2), __ldg(f + 3));
          const uint32_t size = 1u << ins[6];
          if (me)
            for (uint32_t j = 0; j < size; j++) {
              double2 v = AMP(j);
              AMP(j) = cmul(v, ph0);
              AMP(size + j) = cmul(v, ph1);
            }
          break;
        }
        case FS_OP_GAMMA_ROT: {
          const int par = (fx[ins[1]] >> lane) & 1;
          const double* f = P.fparams + ins[5] + 2 * par;
          gamma = cmul(gamma, make_double2(__ldg(f), __ldg(f + 1)));
          break;
        }
        case FS_OP_ARRAY_ROT: {
          const int par = (fx[ins[1]] >> lane) & 1;
          const int a = ins[2];
          const double* f = P.fparams + ins[5];
          const double2 e0 = make_double2(__ldg(f), __ldg(f + 1)), e1 = make_double2(__ldg(f + 2), __ldg(f + 3));
          const double2 ph0 = par ? e1 : e0, ph1 = par ? e0 : e1;
          const uint32_t size = 1u << ins[6];
          if (me)
            for (uint32_t j = 0; j < size; j++) AMP(j) = cmul(AMP(j), ((j >> a) & 1) ? ph1 : ph0);
          break;
        }
        case FS_OP_MEAS_DSTATIC: {
          const int virt = ins[1], rec = ins[3];
          const uint32_t bitw = fx[virt] ^ flipw;
          if (forced) {
            int fo = forced[rec];
            fail(me && fo >= 0 && fo != (int)((bitw >> lane) & 1), FS_ERR_SHOT_FORCED);
          }
          put_record(rec, bitw);
          __syncwarp();
          break;
        }
        case FS_OP_MEAS_DRANDOM: {
          const int virt = ins[1], rec = ins[3];
          const uint32_t pw = fz[virt];
          const int pbit = (pw >> lane) & 1;
          const int fo = forced ? forced[rec] : -1;
          int coin;
          if (SPLITMIX) {
            coin = (fo >= 0) ? (fo ^ pbit ^ (int)(flipw & 1)) : (me ? rng.sm.bit() : 0);
          } else {
            const uint32_t cw = coin_word(A.seed, wabs, ins[2]);
            const int cbit = SEG ? (int)(shot & 31) : lane;
            coin = (fo >= 0) ? (fo ^ pbit ^ (int)(flipw & 1)) : (int)((cw >> cbit) & 1);
          }
          const uint32_t coinw = __ballot_sync(kFull, coin);
          __syncwarp();
          if (lane == 0) {
            uint32_t t = fx[virt];
            fx[virt] = fz[virt] ^ coinw;
            fz[virt] = t;
          }
          gamma = cscale(gamma, kInvSqrt2);
          put_record(rec, coinw ^ pw ^ flipw);
          __syncwarp();
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
            if (lane == 0) {
              const int po = ins[4] >> 8, pc = ins[4] & 0xFF;
              for (int j = 0; j < pc; j++) word_gate(fx, fz, __ldg(P.gates + po + j));
            }
            __syncwarp();
          }
          const int parity = (fx[virt] >> lane) & 1;
          int recbit = 0, brbit = 0;
          bool bad = false;
          int badcode = 0;
          if (me) {
            double p1 = 0.0, p_all = 0.0;
            if (collapse) {
              if (size == 2) {
                double2 a0 = AMP(0), a1 = AMP(1);
                double2 b0 = cadd(cmul(u00, a0), cmul(u01, a1));
                double2 b1 = cadd(cmul(u10, a0), cmul(u11, a1));
                p1 = cnorm2(b1);
                p_all = __dadd_rn(p1, cnorm2(b0));
              } else if (size <= 2 * kSmall) {
                for (uint32_t j = 0; j < half; j++) {
                  uint32_t i0 = ins0(j, a);
                  double2 a0 = AMP(i0), a1 = AMP(i0 + st);
                  double q1 = cnorm2(cadd(cmul(u10, a0), cmul(u11, a1)));
                  double2 b0 = cadd(cmul(u00, a0), cmul(u01, a1));
                  p1 = __dadd_rn(p1, q1);
                  p_all = __dadd_rn(p_all, __dadd_rn(q1, cnorm2(b0)));
                }
              } else {
                for (uint32_t j = 0; j < half; j++) {
                  uint32_t i0 = ins0(j, a);
                  p1 = __dadd_rn(p1, cnorm2(cadd(cmul(AMP(i0), u10), cmul(u11, AMP(i0 + st)))));
                }
                for (uint32_t j = 0; j < size; j++) p_all = __dadd_rn(p_all, cnorm2(AMP(j)));
              }
              if (p1 != p1) { bad = true; badcode = FS_ERR_SHOT_NAN; }
              p1 = p_all > 0 ? __ddiv_rn(p1, p_all) : 0.0;
            } else {
              if (size == 2) p1 = cnorm2(AMP(1));
              else
                for (uint32_t j = 0; j < half; j++) p1 = __dadd_rn(p1, cnorm2(AMP(ins0(j, a) | st)));
              if (p1 != p1) { bad = true; badcode = FS_ERR_SHOT_NAN; }
              if (!renorm) {
                double norm2 = 0.0;
                for (uint32_t j = 0; j < size; j++) norm2 = __dadd_rn(norm2, cnorm2(AMP(j)));
                p1 = norm2 > 0 ? __ddiv_rn(p1, norm2) : 0.0;
              }
            }
            if (!bad) {
              if (p1 < 0.0) p1 = 0.0;
              else if (p1 > 1.0) p1 = 1.0;
              const int fo = forced ? forced[rec] : -1;
              double pb;
              if (fo < 0) {
                rng.begin(i, TAG_BORN);
                brbit = rng.uniform() < p1 ? 1 : 0;
                pb = brbit ? p1 : __dsub_rn(1.0, p1);
                if (pb < kBranchFloor) { brbit ^= 1; pb = __dsub_rn(1.0, pb); }
              } else {
                brbit = fo ^ parity ^ FS_FLIP(I0.x);
                pb = brbit ? p1 : __dsub_rn(1.0, p1);
                if (pb < kBranchFloor) { bad = true; badcode = FS_ERR_SHOT_FORCED; }
              }
              if (!bad) {
                recbit = brbit ^ parity ^ FS_FLIP(I0.x);
                if (collapse) {
                  const double scale = renorm ? __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(pb, p_all))) : 1.0;
                  const double2 k0 = brbit == 0 ? cscale(u00, scale) : cscale(u10, scale);
                  const double2 k1 = brbit == 0 ? cscale(u01, scale) : cscale(u11, scale);
                  for (uint32_t j = 0; j < half; j++) {
                    uint32_t i0 = ins0(j, a);
                    AMP(j) = cadd(cmul(k0, AMP(i0)), cmul(k1, AMP(i0 + st)));
                  }
                } else {
                  const double scale = renorm ? __ddiv_rn(1.0, __dsqrt_rn(pb)) : 1.0;
                  const uint32_t dead = 1u - brbit;
                  for (uint32_t j = 0; j < size; j++) {
                    if (((j >> a) & 1) == dead) AMP(j) = make_double2(0.0, 0.0);
                    else if (renorm) AMP(j) = cscale(AMP(j), scale);
                  }
                }
                if (renorm) gamma = cscale(gamma, __dsqrt_rn(pb));
              }
            }
          }
          fail(bad, badcode);
          branch = brbit;
          const uint32_t recw = __ballot_sync(kFull, recbit);
          if (collapse) {
            const uint32_t brw = __ballot_sync(kFull, brbit);
            if (lane == 0) fx[virt] ^= brw;
          }
          put_record(rec, recw);
          __syncwarp();
          break;
        }
        case FS_OP_RETIRE: {
          const int virt = ins[1], a = ins[2];
          const uint32_t half = (1u << ins[6]) >> 1;
          if (me)
            for (uint32_t j = 0; j < half; j++) AMP(j) = AMP(ins0(j, a) + ((uint32_t)branch << a));
          const uint32_t brw = __ballot_sync(kFull, me && branch);
          if (lane == 0) fx[virt] ^= brw;
          __syncwarp();
          break;
        }
        case FS_OP_COND_FRAME: {
          const uint32_t rw = slots[__ldg(P.bit_slot + ins[3])];
          if (lane == 0 && rw) xor_paulis<false>(P, fx, fz, ins[1], ins[2], rw);
          __syncwarp();
          break;
        }
        case FS_OP_NOISE: {
          if (fmodes) {
            if (me) {
              ShotDraws& d = rng;
              d.begin(i, TAG_FORCED);
              forced_faults_shot(P, fx, fz, lanebit, ins, fmodes, d, 1, true);
            }
          } else if (SPLITMIX) {
            if (me) hazard_shot(P, fx, fz, lanebit, ins, rng.sm);
          } else if (SEG) {
            if (me) {  // own word's generator; keep only this shot's faults
              const int hi = ins[2], mylane = (int)(shot & 31);
              for (;;) {
                if (pend_site < 0) {
                  int st_, ln_, cs_;
                  const int r = lgen.step(P, st_, ln_, cs_);
                  if (r == 2) { pend_site = 0x7FFFFFFF; break; }
                  if (r == 0) continue;
                  pend_site = st_; pend_lane = ln_; pend_case = cs_;
                }
                if (pend_site >= hi) break;
                if (pend_lane == mylane) xor_case_strided(P, fx, fz, pend_case, lanebit, 1, true);
                pend_site = -1;
              }
            }
          } else if (lane == 0) {
            fbuf.apply_until(P, ins[2], [&](int c, int l) {
              const int off = __ldg(P.case_pauli_off + c), end = __ldg(P.case_pauli_off + c + 1);
              for (int j = off; j < end; j++) {
                const uint32_t e = __ldg(P.paulis + j);
                (FS_PAULI_Z(e) ? fz : fx)[FS_PAULI_Q(e)] ^= 1u << l;
              }
            });
          }
          __syncwarp();
          break;
        }
        case FS_OP_DETECTOR:
        case FS_OP_OBSERVABLE: {
          uint32_t wv = 0;
          for (int j = 0; j < ins[3]; j++) wv ^= slots[__ldg(P.bit_slot + __ldg(P.reclists + ins[2] + j))];
          __syncwarp();
          if (op == FS_OP_DETECTOR) {
            put_out(A.det + (size_t)ins[1] * A.W, wv);
            if (lane == 0) {
              const int sl = __ldg(P.bit_slot + P.R + ins[1]);
              if (sl >= 0) slots[sl] = wv;
            }
          } else if (lane == 0) {
            obsw[ins[1]] ^= wv & alive;
          }
          __syncwarp();
          break;
        }
        case FS_OP_POSTSELECT: {
          const int bid = ins[1] == 0 ? P.R + ins[2] : ins[2];
          const uint32_t bw = slots[__ldg(P.bit_slot + bid)];
          const uint32_t rej = (bw ^ (ins[3] ? kFull : 0u)) & alive;
          alive &= ~rej;
          if (rej && (A.t_fx || A.t_gamma || A.t_amps || A.t_draws)) {
            dump_trace(rej, i);
            dumped |= rej;
          }
          break;
        }
        default: break;
      }
    }
    __syncwarp();
    while (cpi < A.ncp && __ldg(A.cp_at + cpi) == i_end) dump_cp(cpi++);
    if (!SEG) {
      if (lane == 0) {
        for (int o = 0; o < P.O; o++) A.obs[(size_t)o * A.W + w] = obsw[o] & validmask;
        A.accepted[w] = alive & validmask;
        A.error[w] = errmask;
        if (errmask) atomicMax(A.status, errcode);
      }
      dump_trace(validmask & ~dumped, stop);
    } else {
      // shots that ended in this segment (halted, errored, or the program finished)
      const uint32_t ended = S.last ? validmask : (validmask & ~alive);
      if ((ended >> lane) & 1) {
        for (int o = 0; o < P.O; o++)
          if ((obsw[o] >> lane) & 1) atomicOr(A.obs + (size_t)o * A.W + (si >> 5), 1u << (si & 31));
        if ((alive >> lane) & 1) atomicOr(A.accepted + (si >> 5), 1u << (si & 31));
        if ((errmask >> lane) & 1) atomicOr(A.error + (si >> 5), 1u << (si & 31));
      }
      if (lane == 0 && errmask) atomicMax(A.status, errcode);
      if (A.t_fx || A.t_gamma || A.t_amps || A.t_draws) dump_trace(ended & ~dumped, S.last ? stop : i_end);
      if (!S.last) {  // compact the survivors into the output store
        const uint32_t surv = alive & validmask;
        uint32_t base = 0;
        if (lane == 0 && surv) base = atomicAdd(S.n_out, (uint32_t)__popc(surv));
        base = __shfl_sync(kFull, base, 0);
        if ((surv >> lane) & 1) {
          const uint32_t slot = base + __popc(surv & ((1u << lane) - 1u));
          const StateStore& O = S.out;
          O.shot[slot] = (uint32_t)si;
          for (int j = 0; j < S.nfw; j++) {
            uint32_t v = 0;
            for (int b = 32 * j; b < 32 * j + 32 && b < 2 * P.n; b++)
              v |= (((b < P.n ? fx[b] : fz[b - P.n]) >> lane) & 1u) << (b & 31);
            O.frame[(size_t)slot * S.nfw + j] = v;
          }
          for (int j = 0; j < S.nsw; j++) {
            uint32_t v = 0;
            for (int b = 32 * j; b < 32 * j + 32 && b < P.num_slots; b++) v |= ((slots[b] >> lane) & 1u) << (b & 31);
            O.slotbits[(size_t)slot * S.nsw + j] = v;
          }
          for (int j = 0; j < S.now; j++) {
            uint32_t v = 0;
            for (int b = 32 * j; b < 32 * j + 32 && b < P.O; b++) v |= ((obsw[b] >> lane) & 1u) << (b & 31);
            O.obsbits[(size_t)slot * S.now + j] = v;
          }
          O.gamma[slot] = gamma;
          if (SPLITMIX) O.smcount[slot] = rng.sm.count;
          else {
            uint32_t* gi = O.gen_i + (size_t)slot * 6;
            gi[0] = lgen.step_no; gi[1] = (uint32_t)lgen.run; gi[2] = (uint32_t)lgen.cl;
            gi[3] = (uint32_t)pend_site; gi[4] = (uint32_t)pend_lane; gi[5] = (uint32_t)pend_case;
            O.gen_c[slot] = lgen.c;
          }
          const uint32_t sz = 1u << S.k_out;
          for (uint32_t j = 0; j < sz; j++) O.amps[store_amp_index(slot, j, sz, O.shot_major)] = AMP(j);
        }
      }
    }
    __syncwarp();
  }
#undef AMP
}

}  // namespace fs
