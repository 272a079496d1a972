// fs_sampler.cu -- C ABI (include/fs_sampler.h) over the sm_100a engines.
//
//   engine 1 (fs_frame.cuh)   frame-only programs: lane = 32-shot word, 1024 shots per warp
//   engine 0 (fs_general.cuh) everything else: warp = 32-shot word, lane = shot
//
// No CPU fallback exists: if CUDA is unavailable every entry point fails with FS_ERR_CUDA.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "fs_frame.cuh"
#include "fs_general.cuh"
#include "fs_hbm.cuh"
#include "fs_hbm_fused.cuh"
#include "fs_block.cuh"
#include "fs_jit.cuh"
#include "fs_affine.cuh"
#include "fs_jit_kernels.cuh"
#include "fs_format.cuh"
#include "fs_stratum.cuh"

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define FS_CUDA_TRY(expr)                                                                  \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return set_error(FS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

constexpr size_t kSmemBudget = 200 * 1024;  // per block, leaves room for L1
constexpr size_t kAffSmemBudget = 224 * 1024;  // affine frame kernel: row buffers of one block per SM

// every entry point runs on the device the program was created on (its allocations and NVRTC
// modules live in that device's primary context), whatever device the calling thread has current
struct DeviceGuard {
  int prev = -1, want;
  explicit DeviceGuard(int dev) : want(dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != want) cudaSetDevice(want);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Stage {  // carve-out of one device allocation
  size_t off = 0;
  unsigned char* base = nullptr;
  template <class T>
  T* take(size_t count) {
    if (!count) return nullptr;
    T* r = reinterpret_cast<T*>(base + off);
    off = align_up(off + count * sizeof(T), 256);
    return r;
  }
};

}  // namespace

struct HbmStep {
  enum Kind { SCALAR, ARR, PASS, MEAS, DUMP } kind;
  int i0, i1;
  int cp;               // DUMP: checkpoint index
  fs::DevAxisMap map;   // DUMP: logical -> physical axes at the checkpoint
  fs::ArrOp op;
  uint64_t count;
  int pass;
  int collapse;
  double2 u10, u11;
};

struct HbmPlan {
  bool built = false, fused = false;
  int stop = -1;
  std::vector<int> cuts;               // checkpoints (instruction counts) the plan dumps at
  std::vector<HbmStep> steps;
  std::vector<fs::PassDesc> passes;
  std::vector<fs::TileOp> tileops;
  std::vector<uint32_t> code;          // pass microcode (fs_hbm_fused.cuh)
  std::vector<fs::PassConst> consts;
  std::vector<int> final_live;
};

namespace {
constexpr int kLargeK = 16;  // k_max at which active arrays move to the HBM engine
constexpr int kBlockK = 9;   // segment active dimension at which a shot gets a whole CTA (or warp); measured on config 4: lane-per-shot 2.4x faster at k = 7, 2.6x slower at k = 10
constexpr int kChunks = 4;   // max word chunks of the fault-list | frame-kernel pipeline; default 1 (2-4 measured 10-27 % slower), FS_JIT_CHUNKS overrides
}  // namespace

// testing / experiment switches, read once at fs_program_create (never on a launch path)
struct EnvSwitches {
  bool no_affine = false;      // FS_NO_AFFINE: frame-only programs use the fault-list frame kernel
  bool block_no_jit = false;   // FS_BLOCK_NO_JIT: segmented engine interprets every segment
  bool block_no_wjit = false;  // FS_BLOCK_NO_WJIT: no packed-frame segment kernels (fs_wseg.cuh): warp-per-shot segments keep the interpreter, CTA-per-shot ones the shared-VM specialised form
  bool seg_no_ljit = false;    // FS_SEG_NO_LJIT: lane-per-shot segments keep the interpreter (no fs_lseg.cuh kernels)
  bool block_no_fuse = false;  // FS_BLOCK_NO_FUSE: block engine runs ArrayGates one sweep each (no star groups)
  int block_k = 0;             // FS_BLOCK_K: segment k at which a shot gets a warp / CTA (0 = default)
  bool hbm_fused = false;      // FS_HBM_FUSED: fused tile passes also under FS_FORCE_HBM
  bool hbm_unfused = false;    // FS_HBM_UNFUSED: per-instruction large-k kernels only
  bool hbm_no_jit = false;     // FS_HBM_NO_JIT: pass microcode interpreter instead of fs_pass_<i>
  bool pass_tma = false;       // FS_PASS_TMA: fs_pass_<i> stage tiles with TMA bulk copies instead of cp.async
  int jit_chunks = 1;          // FS_JIT_CHUNKS: fault-list | frame-kernel pipeline depth
  uint64_t stratum_chunk = 0;  // FS_STRATUM_CHUNK: stratified-sampling chunk (tests)
  void read() {
    no_affine = getenv("FS_NO_AFFINE") != nullptr;
    block_no_jit = getenv("FS_BLOCK_NO_JIT") != nullptr;
    block_no_fuse = getenv("FS_BLOCK_NO_FUSE") != nullptr;
    block_no_wjit = getenv("FS_BLOCK_NO_WJIT") != nullptr;
    seg_no_ljit = getenv("FS_SEG_NO_LJIT") != nullptr;
    if (const char* e = getenv("FS_BLOCK_K")) block_k = std::max(1, atoi(e));
    hbm_fused = getenv("FS_HBM_FUSED") != nullptr;
    hbm_unfused = getenv("FS_HBM_UNFUSED") != nullptr;
    hbm_no_jit = getenv("FS_HBM_NO_JIT") != nullptr;
    pass_tma = getenv("FS_PASS_TMA") != nullptr;
    if (const char* e = getenv("FS_JIT_CHUNKS")) jit_chunks = std::max(1, std::min(kChunks, atoi(e)));
    if (const char* e = getenv("FS_STRATUM_CHUNK")) stratum_chunk = std::max<uint64_t>(32, (uint64_t)atoll(e) / 32 * 32);
  }
};

struct fs_prog {
  fs_prog_desc desc;  // scalar fields only (pointers refer to host memory of the creator)
  EnvSwitches env;
  fs::DevProg dp;
  void* dbuf = nullptr;
  int device = 0;
  int num_sms = 0;
  std::mutex mu;
  // general engine scratch (per resident warp) and call-local buffers
  double2* scratch = nullptr;
  size_t scratch_bytes = 0;
  int* d_status = nullptr;
  // host-API staging
  void* stage = nullptr;
  size_t stage_bytes = 0;
  int64_t* d_counts = nullptr;
  size_t counts_len = 0;
  // host copies used by the large-k engine's host-side walk and the JIT generator
  std::vector<int32_t> h_instrs, h_sched;
  std::vector<double> h_fparams;
  std::vector<uint32_t> h_gates, h_paulis;
  std::vector<int32_t> h_reclists, h_record_out, h_bit_slot, h_plans, h_case_pauli_off, h_site_case_off;
  std::vector<double> h_site_prob, h_case_cum;
  // program-specialised frame kernel (fs_jit.cuh); built on first use
  int jit_state = 0;  // 0 not tried, 1 ready, -1 failed (interpreter is used)
  std::string jit_error;
  fsjit::Compiled jit;
  uint16_t* d_pslot = nullptr;
  int jit_nslots = 0;
  void* flist = nullptr;  // per-word fault lists for the specialised kernel
  size_t flist_bytes = 0;
  uint32_t flist_cap = 0;
  int* d_site_block = nullptr;  // flip geometry: block_hi | row_off | block_cap
  int jit_nblocks = 0;
  int jit_stage = fsjit::kJitStage;
  // affine frame kernel (fs_affine.cuh): 0 not tried, 1 ready, -1 not applicable / failed
  int aff_state = 0;
  std::string aff_error;
  fsjit::Compiled aff;
  uint32_t* d_aff_tables = nullptr;
  int aff_threads = 0, aff_rows = 0, aff_occ = 0, gjit_occ = 0;
  size_t aff_smem = 0;
  // stratified sampling: suffix Poisson-binomial table of stratum w, per-chunk modes + outputs
  int strat_w = -1;
  double strat_weight = 0.0;
  double* d_strat = nullptr;
  void* strat_buf = nullptr;
  size_t strat_bytes = 0;
  // fs_format scratch (kept flags, ranks, lengths, offsets, scan temp, weight text)
  void* fmt = nullptr;
  size_t fmt_bytes = 0;
  // instrumentation: kernel launch count, optional events around the dominant kernel's launches
  uint64_t launches = 0;
  bool ktimer = false;
  std::vector<cudaEvent_t> kev;
  size_t kev_n = 0;  // fault-list capacity per word (frame kernel: its smem stage)
  int flip_rows = 0, flip_capmax = 0;
  int gjit_threads = 128;
  cudaStream_t aux = nullptr;  // fault-list generation overlapped with the specialised kernels
  cudaEvent_t ev[kChunks + 1] = {};
  size_t gjit_smem = 0;
  // segmented general engine: ping-pong survivor state stores
  void* seg_pool[2] = {nullptr, nullptr};
  std::vector<uint32_t> seg_counts;  // diagnostics: shots entering each segment (per chunk)
  size_t seg_bytes[2] = {0, 0};
  // large-k engine state
  HbmPlan hplan;
  fs::PassDesc* d_passes = nullptr;
  fs::TileOp* d_tileops = nullptr;
  uint32_t* d_code = nullptr;
  fs::PassConst* d_consts = nullptr;
  // program-specialised pass kernels (NVRTC) of the current plan: 0 = not built, 1 = ready, -1 = failed
  int pass_jit = 0;
  std::vector<fsjit::CUfunction> pass_fn;
  std::string pass_jit_err;
  // program-specialised segment kernels of the block engine (key: segment begin), Philox stream
  int seg_jit = 0;
  std::map<int, int> seg_G;  // block segments in the packed-frame form (fs_wseg.cuh): threads per shot
  std::set<int> seg_lane;  // segment starts compiled as lane-per-shot kernels (fs_lseg.cuh)
  std::map<int, int> seg_occ;  // resident blocks per SM of the specialised segment kernels
  std::vector<int32_t> h_next_array, h_frame_mat_off, h_fuse_at, h_fuse;
  std::map<int, fsjit::CUfunction> seg_fn;
  std::string seg_jit_err;
  void* d_cp = nullptr;  // checkpoint instruction counts + amplitude offsets of the current call
  size_t cp_bytes = 0;
  std::vector<int> cp_list;        // the current call's checkpoints (host copy, large-k planner)
  std::vector<uint64_t> cp_offs;   // their amplitude offsets (complex elements)
  void* hbm = nullptr;
  size_t hbm_bytes = 0;
  uint64_t hbm_B = 0;
};


extern "C" int fs_abi_version(void) { return FS_ABI_VERSION; }
extern "C" const char* fs_last_error(void) { return g_last_error.c_str(); }

extern "C" int fs_program_create(const fs_prog_desc* d, fs_prog** out) {
  if (!d || !out) return set_error(FS_ERR_ARG, "null argument");
  if (d->abi_version != FS_ABI_VERSION) return set_error(FS_ERR_ARG, "ABI version mismatch");
  if (d->n < 0 || d->n >= (1 << 14) || d->k_max < 0 || d->k_max > 30 || d->num_instrs < 0)
    return set_error(FS_ERR_ARG, "program dimensions out of range");
  int dev = 0;
  FS_CUDA_TRY(cudaGetDevice(&dev));
  auto* p = new fs_prog();
  p->desc = *d;
  p->device = dev;
  p->env.read();
  FS_CUDA_TRY(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev));

  // pack every table into one device allocation (16 B aligned sections)
  struct Sec { const void* src; size_t bytes; size_t off; };
  std::vector<Sec> secs;
  size_t total = 0;
  auto add = [&](const void* src, size_t bytes) {
    size_t off = total;
    secs.push_back({src, bytes, off});
    total = align_up(total + std::max<size_t>(bytes, 16), 16);
    return off;
  };
  const int E = d->num_sites, R = d->record_count, D = d->num_detectors;
  size_t o_instrs = add(d->instrs, sizeof(int32_t) * FS_INS_WORDS * d->num_instrs);
  size_t o_sched = add(d->schedule, sizeof(int32_t) * d->num_instrs);
  size_t o_fp = add(d->fparams, sizeof(double) * d->num_fparams);
  size_t o_gates = add(d->gates, sizeof(uint32_t) * d->num_gates);
  size_t o_paulis = add(d->paulis, sizeof(uint32_t) * d->num_paulis);
  size_t o_rl = add(d->reclists, sizeof(int32_t) * d->num_reclists);
  size_t o_sp = add(d->site_prob, sizeof(double) * E);
  size_t o_sco = add(d->site_case_off, sizeof(int32_t) * (E + 1));
  size_t o_cc = add(d->case_cum, sizeof(double) * d->num_cases);
  size_t o_cpo = add(d->case_pauli_off, sizeof(int32_t) * (d->num_cases + 1));
  size_t o_ch = add(d->cum_hazard, sizeof(double) * (E + 1));
  size_t o_pl = add(d->plans, sizeof(int32_t) * 2 * d->num_plans);
  size_t o_ro = add(d->record_out, sizeof(int32_t) * R);
  size_t o_bs = add(d->bit_slot, sizeof(int32_t) * (R + D));
  // Philox noise runs: consecutive sites whose probabilities agree to 1e-9
  // (relative) share one geometric process at q = max p, thinned by p/q per candidate; certain
  // sites (p >= 1) are single runs; p = 0 / caseless sites never fire
  std::vector<int32_t> run_start, run_len;
  std::vector<double> run_lp, run_q;
  for (int site = 0; site < E;) {
    const double prob = d->site_prob[site];
    const int nc = d->site_case_off[site + 1] - d->site_case_off[site];
    if (!(prob > 0.0) || nc == 0) { site++; continue; }
    if (prob >= 1.0) {
      run_start.push_back(site); run_len.push_back(0); run_lp.push_back(0.0); run_q.push_back(1.0);
      site++;
      continue;
    }
    int len = 1;
    double lo = prob, hi = prob;
    while (site + len < E) {
      const double pn = d->site_prob[site + len];
      if (!(pn > 0.0) || pn >= 1.0 || d->site_case_off[site + len + 1] - d->site_case_off[site + len] == 0) break;
      const double nlo = std::min(pn, lo), nhi = std::max(pn, hi);
      if (!(nhi <= nlo * (1.0 + 1e-9))) break;
      lo = nlo; hi = nhi; len++;
    }
    run_start.push_back(site); run_len.push_back(len); run_lp.push_back(1.0 / log1p(-hi)); run_q.push_back(hi);
    site += len;
  }
  const int nruns = (int)run_start.size();
  size_t o_rs = add(run_start.data(), sizeof(int32_t) * nruns);
  size_t o_rl2 = add(run_len.data(), sizeof(int32_t) * nruns);
  size_t o_rlp = add(run_lp.data(), sizeof(double) * nruns);
  size_t o_rq = add(run_q.data(), sizeof(double) * nruns);
  // FrameGates as GF(2) matrices for the block engine (a warp applies one with ballots + popcounts
  // instead of thread 0 walking the gate list): column j = the gate list applied to basis bit j
  const int n2 = 2 * d->n;
  const bool mats = n2 <= 128 && d->k_max > 0;
  std::vector<uint32_t> frame_mat;
  std::vector<int32_t> frame_mat_off(d->num_instrs + 1, -1);
  // one frame gate on a 0/1 vector (fx = v, fz = v + n)
  auto frame_gate = [&](uint32_t* fx, uint32_t* fz, int g, int a, int b) {
    uint32_t tt;
    switch (g) {
      case FS_G_H: tt = fx[a]; fx[a] = fz[a]; fz[a] = tt; break;
      case FS_G_S: case FS_G_SDAG: fz[a] ^= fx[a]; break;
      case FS_G_CX: fx[b] ^= fx[a]; fz[a] ^= fz[b]; break;
      case FS_G_CZ: fz[b] ^= fx[a]; fz[a] ^= fx[b]; break;
      case FS_G_SWAP:
        tt = fx[a]; fx[a] = fx[b]; fx[b] = tt;
        tt = fz[a]; fz[a] = fz[b]; fz[b] = tt;
        break;
      default: break;
    }
  };
  // the frame action of instructions [i0, i1) (FrameGates lists and the frame side of ArrayGates)
  // as one matrix appended to frame_mat; returns its word offset
  auto build_matrix = [&](int i0, int i1) {
    const int32_t off = (int32_t)frame_mat.size();
    frame_mat.resize(frame_mat.size() + (size_t)n2 * 4, 0u);
    std::vector<uint32_t> v(n2);
    for (int j = 0; j < n2; j++) {
      std::fill(v.begin(), v.end(), 0u);
      v[j] = 1u;
      for (int i = i0; i < i1; i++) {
        const int* I = d->instrs + (size_t)i * FS_INS_WORDS;
        const int op = FS_OPCODE(I[0]);
        if (op == FS_OP_FRAME) {
          for (int t = 0; t < I[2]; t++) {
            const uint32_t g = d->gates[I[1] + t];
            frame_gate(v.data(), v.data() + d->n, FS_GATE_G(g), FS_GATE_A(g), FS_GATE_B(g));
          }
        } else if (op == FS_OP_ARRAY_GATE) {
          frame_gate(v.data(), v.data() + d->n, I[1], I[2], I[3]);
        }
      }
      uint32_t* M = frame_mat.data() + off;
      for (int r = 0; r < n2; r++)
        if (v[r] & 1u) M[(size_t)r * 4 + (j >> 5)] |= 1u << (j & 31);
    }
    return off;
  };
  if (mats)
    for (int i = 0; i < d->num_instrs; i++)
      if (FS_OPCODE(d->instrs[(size_t)i * FS_INS_WORDS]) == FS_OP_FRAME) frame_mat_off[i] = build_matrix(i, i + 1);
  // Star groups (block engine): a run of ArrayGates that all act through one pivot axis a --
  // CX(a, b), CZ(a, c), S / S_DAG(a), then at most one H(a) -- with FrameGates in between and an
  // optional closing ArrayRot is one sweep: elements with bit a clear keep their place, element j
  // with bit a set becomes i^(ns + 2 (parity(j & Mz) ^ s0)) * old[j ^ M]; then the H butterfly on
  // a and the ArrayRot phases.  The same values as the per-instruction sweeps (permutations, sign
  // flips and multiplications by +-i are exact), one pass over the array instead of one per gate.
  // Descriptor (8 words): len, a | k << 8, M, Mz, power | hasH << 2 | hasAR << 3,
  // ar_virt | ar_axis << 16, ar_fp, frame matrix offset.
  std::vector<int32_t> fuse_at(d->num_instrs + 1, -1), fuse;
  if (mats && !p->env.block_no_fuse) {
    for (int i = 0; i < d->num_instrs;) {
      const int* I0 = d->instrs + (size_t)i * FS_INS_WORDS;
      if (FS_OPCODE(I0[0]) != FS_OP_ARRAY_GATE) { i++; continue; }
      int pivot = -1, narr = 0, end = i, ar = -1;
      uint32_t M = 0, Mz = 0, ns = 0;
      bool hasH = false;
      std::vector<std::pair<int, uint32_t>> czs;  // (other axis, M at that time)
      const int k = I0[6];
      for (int t = i; t < d->num_instrs; t++) {
        const int* I = d->instrs + (size_t)t * FS_INS_WORDS;
        const int op = FS_OPCODE(I[0]);
        if (op == FS_OP_FRAME) continue;  // absorbed if an array instruction of the group follows
        if (op == FS_OP_ARRAY_ROT) {
          if (I[6] == k && narr > 0) { ar = t; end = t + 1; narr++; }
          break;
        }
        if (op != FS_OP_ARRAY_GATE || I[6] != k || hasH) break;
        const int g = I[1], a = I[4], b = I[5];
        bool ok = true;
        if (g == FS_G_S || g == FS_G_SDAG || g == FS_G_H) {
          if (pivot < 0) pivot = a;
          if (a != pivot) ok = false;
          else if (g == FS_G_H) hasH = true;
          else ns = (ns + (g == FS_G_S ? 1u : 3u)) & 3u;
        } else if (g == FS_G_CX) {
          if (pivot < 0) pivot = a;
          if (a != pivot || b == pivot) ok = false;
          else M ^= 1u << b;
        } else if (g == FS_G_CZ) {
          if (pivot < 0) pivot = a;
          const int other = a == pivot ? b : (b == pivot ? a : -1);
          if (other < 0 || other == pivot) ok = false;
          else { Mz ^= 1u << other; czs.push_back({other, M}); }
        } else {
          ok = false;
        }
        if (!ok) break;
        narr++;
        end = t + 1;
      }
      if (narr < 2) { i++; continue; }
      uint32_t s0 = 0;
      for (auto& cz : czs) s0 ^= ((M ^ cz.second) >> cz.first) & 1u;
      const int* IA = ar >= 0 ? d->instrs + (size_t)ar * FS_INS_WORDS : nullptr;
      fuse_at[i] = (int32_t)(fuse.size() / 8);
      fuse.push_back(end - i);
      fuse.push_back(pivot | (k << 8));
      fuse.push_back((int32_t)M);
      fuse.push_back((int32_t)Mz);
      fuse.push_back((int32_t)(((ns + 2u * s0) & 3u) | (hasH ? 4u : 0u) | (ar >= 0 ? 8u : 0u)));
      fuse.push_back(IA ? (IA[1] | (IA[2] << 16)) : 0);
      fuse.push_back(IA ? IA[5] : 0);
      fuse.push_back(build_matrix(i, end));
      i = end;
    }
  }
  if (fuse.empty()) fuse.assign(8, 0);
  // per-case frame masks (x_q at bit q, z_q at bit n + q) for the packed-frame segment kernels
  std::vector<uint32_t> case_mask;
  if (mats && d->num_cases > 0) {
    case_mask.assign((size_t)4 * d->num_cases, 0u);
    for (int c = 0; c < d->num_cases; c++)
      for (int j = d->case_pauli_off[c]; j < d->case_pauli_off[c + 1]; j++) {
        const uint32_t en = d->paulis[j];
        const int bit = FS_PAULI_Z(en) ? d->n + (int)FS_PAULI_Q(en) : (int)FS_PAULI_Q(en);
        case_mask[(size_t)4 * c + (bit >> 5)] ^= 1u << (bit & 31);
      }
  }
  const bool have_masks = mats;
  if (case_mask.empty()) case_mask.assign(4, 0u);
  if (frame_mat.empty()) frame_mat.push_back(0u);
  size_t o_fm = add(frame_mat.data(), sizeof(uint32_t) * frame_mat.size());
  size_t o_fmo = add(frame_mat_off.data(), sizeof(int32_t) * frame_mat_off.size());
  size_t o_fat = add(fuse_at.data(), sizeof(int32_t) * fuse_at.size());
  size_t o_fus = add(fuse.data(), sizeof(int32_t) * fuse.size());
  size_t o_cm = add(case_mask.data(), sizeof(uint32_t) * case_mask.size());
  std::vector<int32_t> next_array(d->num_instrs + 1, d->num_instrs);
  for (int i = d->num_instrs - 1; i >= 0; i--) {
    const int op = FS_OPCODE(d->instrs[(size_t)i * FS_INS_WORDS]);
    const bool arr = op == FS_OP_ARRAY_GATE || op == FS_OP_EXPAND || op == FS_OP_ARRAY_ROT ||
                     op == FS_OP_MEAS_ACTIVE || op == FS_OP_MEAS_COLLAPSE || op == FS_OP_RETIRE ||
                     (op == FS_OP_FRAME && frame_mat_off[i] >= 0);
    next_array[i] = arr ? i : next_array[i + 1];
  }
  size_t o_na = add(next_array.data(), sizeof(int32_t) * next_array.size());
  std::vector<unsigned char> host(total, 0);
  for (auto& s : secs)
    if (s.src && s.bytes) std::memcpy(host.data() + s.off, s.src, s.bytes);
  cudaError_t e = cudaMalloc(&p->dbuf, total);
  if (e == cudaSuccess) e = cudaMemcpy(p->dbuf, host.data(), total, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_status, sizeof(int));
  if (e != cudaSuccess) {
    delete p;
    return set_error(FS_ERR_CUDA, std::string("program upload: ") + cudaGetErrorString(e));
  }
  auto* b = static_cast<unsigned char*>(p->dbuf);
  fs::DevProg& dp = p->dp;
  dp.n = d->n; dp.k_max = d->k_max; dp.num_instrs = d->num_instrs; dp.R = R;
  dp.U = d->num_user_records; dp.D = D; dp.O = d->num_observables; dp.E = E;
  dp.num_slots = d->num_slots;
  dp.has_psel = 0;
  for (int i = 0; i < d->num_instrs; i++)
    if (FS_OPCODE(d->instrs[i * FS_INS_WORDS]) == FS_OP_POSTSELECT) dp.has_psel = 1;
  dp.instrs = reinterpret_cast<const int*>(b + o_instrs);
  dp.schedule = reinterpret_cast<const int*>(b + o_sched);
  dp.fparams = reinterpret_cast<const double*>(b + o_fp);
  dp.gates = reinterpret_cast<const uint32_t*>(b + o_gates);
  dp.paulis = reinterpret_cast<const uint32_t*>(b + o_paulis);
  dp.reclists = reinterpret_cast<const int*>(b + o_rl);
  dp.site_prob = reinterpret_cast<const double*>(b + o_sp);
  dp.site_case_off = reinterpret_cast<const int*>(b + o_sco);
  dp.case_cum = reinterpret_cast<const double*>(b + o_cc);
  dp.case_pauli_off = reinterpret_cast<const int*>(b + o_cpo);
  dp.cum_hazard = reinterpret_cast<const double*>(b + o_ch);
  dp.plans = reinterpret_cast<const int*>(b + o_pl);
  dp.record_out = reinterpret_cast<const int*>(b + o_ro);
  dp.bit_slot = reinterpret_cast<const int*>(b + o_bs);
  dp.num_runs = nruns;
  dp.run_start = reinterpret_cast<const int*>(b + o_rs);
  dp.run_len = reinterpret_cast<const int*>(b + o_rl2);
  dp.run_lp = reinterpret_cast<const double*>(b + o_rlp);
  dp.run_q = reinterpret_cast<const double*>(b + o_rq);
  dp.next_array = reinterpret_cast<const int*>(b + o_na);
  dp.frame_mat = reinterpret_cast<const uint32_t*>(b + o_fm);
  p->h_next_array = next_array;
  p->h_frame_mat_off = frame_mat_off;
  dp.frame_mat_off = reinterpret_cast<const int*>(b + o_fmo);
  dp.fuse_at = reinterpret_cast<const int*>(b + o_fat);
  dp.fuse = reinterpret_cast<const int*>(b + o_fus);
  dp.case_mask = have_masks ? reinterpret_cast<const uint4*>(b + o_cm) : nullptr;
  p->h_fuse_at = fuse_at;
  p->h_fuse = fuse;
  p->h_instrs.assign(d->instrs, d->instrs + (size_t)FS_INS_WORDS * d->num_instrs);
  p->h_sched.assign(d->schedule, d->schedule + d->num_instrs);
  if (d->num_fparams) p->h_fparams.assign(d->fparams, d->fparams + d->num_fparams);
  p->h_gates.assign(d->gates, d->gates + d->num_gates);
  p->h_paulis.assign(d->paulis, d->paulis + d->num_paulis);
  p->h_reclists.assign(d->reclists, d->reclists + d->num_reclists);
  p->h_record_out.assign(d->record_out, d->record_out + R);
  p->h_bit_slot.assign(d->bit_slot, d->bit_slot + R + D);
  p->h_plans.assign(d->plans, d->plans + 2 * d->num_plans);
  p->h_case_pauli_off.assign(d->case_pauli_off, d->case_pauli_off + d->num_cases + 1);
  p->h_site_case_off.assign(d->site_case_off, d->site_case_off + E + 1);
  p->h_site_prob.assign(d->site_prob, d->site_prob + E);
  p->h_case_cum.assign(d->case_cum, d->case_cum + d->num_cases);
  // pointers of the creator's arrays are not retained
  p->desc.instrs = nullptr;
  *out = p;
  return FS_OK;
}

extern "C" void fs_program_destroy(fs_prog* p) {
  if (!p) return;
  DeviceGuard dg(p->device);
  cudaFree(p->dbuf);
  cudaFree(p->scratch);
  cudaFree(p->d_status);
  cudaFree(p->stage);
  cudaFree(p->d_counts);
  cudaFree(p->hbm);
  cudaFree(p->d_passes);
  cudaFree(p->d_tileops);
  cudaFree(p->d_code);
  cudaFree(p->d_consts);
  cudaFree(p->seg_pool[0]);
  cudaFree(p->seg_pool[1]);
  cudaFree(p->d_pslot);
  for (auto e : p->kev) cudaEventDestroy(e);
  cudaFree(p->fmt);
  cudaFree(p->d_strat);
  cudaFree(p->strat_buf);
  if (p->aux) {
    cudaStreamDestroy(p->aux);
    for (auto& e : p->ev)
      if (e) cudaEventDestroy(e);
  }
  cudaFree(p->flist);
  cudaFree(p->d_site_block);
  cudaFree(p->d_aff_tables);
  cudaFree(p->d_cp);
  if (p->aff.mod && fsjit::api().ok) fsjit::api().cuModuleUnload(p->aff.mod);
  if (p->jit.mod && fsjit::api().ok) fsjit::api().cuModuleUnload(p->jit.mod);
  delete p;
}

static bool wants_hbm(const fs_prog* p, uint32_t flags) { return p->dp.k_max >= kLargeK || (flags & FS_FORCE_HBM); }

static bool wants_general(const fs_prog* p, uint32_t flags, const fs_trace_in* tin, const fs_trace_out* tout) {
  if (p->dp.k_max > 0) return true;
  if (flags & (FS_RNG_SPLITMIX | FS_FORCE_GENERAL)) return true;
  if (tout && (tout->gamma || tout->amps || tout->draws || tout->records)) return true;
  if (tin && tin->ncheckpoints > 0) return true;
  return false;
}

// Diagnostics (not part of include/fs_sampler.h): measured FP64 FMA throughput of this device,
// the denominator of the on-chip roofline of the small-k configurations (bench.py).
__global__ void fp64_peak_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; i++) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.0) out[0] = a0;
}

extern "C" int fs_debug_fp64_peak(double* tflops) {
  if (!tflops) return FS_ERR_ARG;
  int dev = 0, sms = 0;
  FS_CUDA_TRY(cudaGetDevice(&dev));
  FS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* d = nullptr;
  FS_CUDA_TRY(cudaMalloc(&d, 8));
  const int iters = 1 << 14, threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_peak_kernel<<<blocks, threads>>>(d, iters);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) fp64_peak_kernel<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  FS_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  *tflops = 5.0 * blocks * threads * (double)iters * 8 * 2 / (ms * 1e-3) / 1e12;
  return FS_OK;
}

// Diagnostics (not part of include/fs_sampler.h): source of the program-specialised frame kernel
// and the state of its compilation.  Used by tests/test_host.py to compile the generated
// kernel with NVRTC on a CPU-only host.
extern "C" int fs_debug_jit_source(const fs_prog_desc* d, char* buf, size_t len) {
  if (!d) return -1;
  const int R = d->record_count, D = d->num_detectors, E = d->num_sites;
  std::vector<int32_t> ins(d->instrs, d->instrs + (size_t)FS_INS_WORDS * d->num_instrs);
  std::vector<uint32_t> g(d->gates, d->gates + d->num_gates), pa(d->paulis, d->paulis + d->num_paulis);
  std::vector<int32_t> rl(d->reclists, d->reclists + d->num_reclists), ro(d->record_out, d->record_out + R);
  std::vector<int32_t> bs(d->bit_slot, d->bit_slot + R + D), pl(d->plans, d->plans + 2 * d->num_plans);
  std::vector<int32_t> cpo(d->case_pauli_off, d->case_pauli_off + d->num_cases + 1);
  std::vector<int32_t> sco(d->site_case_off, d->site_case_off + E + 1);
  std::vector<double> sp(d->site_prob, d->site_prob + E);
  fsjit::FrameKernelSource K = fsjit::gen_frame_kernel(*d, ins, g, pa, rl, ro, bs, pl, cpo, sco, sp);
  if (buf && len) {
    size_t m = std::min(len - 1, K.src.size());
    std::memcpy(buf, K.src.data(), m);
    buf[m] = 0;
  }
  return (int)K.src.size();
}

// source of the affine frame kernel (fs_affine.cuh); negative if not applicable
extern "C" int fs_debug_aff_source(const fs_prog_desc* d, char* buf, size_t len) {
  if (!d) return -1;
  const int R = d->record_count, D = d->num_detectors, E = d->num_sites;
  std::vector<int32_t> ins(d->instrs, d->instrs + (size_t)FS_INS_WORDS * d->num_instrs);
  std::vector<uint32_t> g(d->gates, d->gates + d->num_gates), pa(d->paulis, d->paulis + d->num_paulis);
  std::vector<int32_t> rl(d->reclists, d->reclists + d->num_reclists), ro(d->record_out, d->record_out + R);
  std::vector<int32_t> bs(d->bit_slot, d->bit_slot + R + D);
  std::vector<int32_t> cpo(d->case_pauli_off, d->case_pauli_off + d->num_cases + 1);
  std::vector<int32_t> sco(d->site_case_off, d->site_case_off + E + 1);
  std::vector<double> sp(d->site_prob, d->site_prob + E), cc(d->case_cum, d->case_cum + d->num_cases);
  fsjit::AffineKernelSource K = fsjit::gen_affine_frame_kernel(*d, ins, g, pa, rl, ro, bs, cpo, sco, sp, cc, kAffSmemBudget);
  if (!K.why.empty()) return -2;
  if (buf && len) {
    size_t m = std::min(len - 1, K.src.size());
    std::memcpy(buf, K.src.data(), m);
    buf[m] = 0;
  }
  return (int)K.src.size();
}

// segmented engine: shots entering each segment of the last call (chunks concatenated)
extern "C" int fs_debug_seg_counts(fs_prog* p, uint32_t* out, int cap) {
  if (!p) return -1;
  const int n = (int)p->seg_counts.size();
  for (int i = 0; i < n && i < cap; i++) out[i] = p->seg_counts[i];
  return n;
}

// the same generator from a descriptor (no device needed: source inspection / offline SASS checks)
extern "C" int fs_debug_gjit_source_desc(const fs_prog_desc* d, char* buf, size_t len) {
  if (!d) return -1;
  auto vec = [](const auto* ptr, size_t n) { return std::vector<std::remove_cv_t<std::remove_pointer_t<decltype(ptr)>>>(ptr, ptr + n); };
  std::vector<int32_t> ins = vec(d->instrs, (size_t)d->num_instrs * FS_INS_WORDS);
  fsjit::GeneralKernelSource K = fsjit::gen_general_kernel(
      *d, ins, vec(d->gates, d->num_gates), vec(d->paulis, d->num_paulis), vec(d->reclists, d->num_reclists),
      vec(d->record_out, d->record_count), vec(d->bit_slot, d->record_count + d->num_detectors),
      vec(d->case_pauli_off, d->num_cases + 1), vec(d->site_case_off, d->num_sites + 1), vec(d->fparams, d->num_fparams));
  if (buf && len) {
    size_t m = std::min(len - 1, K.src.size());
    std::memcpy(buf, K.src.data(), m);
    buf[m] = 0;
  }
  return (int)K.src.size();
}

extern "C" int fs_debug_gjit_source(fs_prog* p, char* buf, size_t len) {
  if (!p) return -1;
  fsjit::GeneralKernelSource K = fsjit::gen_general_kernel(p->desc, p->h_instrs, p->h_gates, p->h_paulis,
                                                           p->h_reclists, p->h_record_out, p->h_bit_slot,
                                                           p->h_case_pauli_off, p->h_site_case_off, p->h_fparams);
  if (buf && len) {
    size_t m = std::min(len - 1, K.src.size());
    std::memcpy(buf, K.src.data(), m);
    buf[m] = 0;
  }
  return (int)K.src.size();
}

namespace {
int plan_hbm(fs_prog* p, int stop, bool fused, const std::vector<int>& cuts = {});
}
// large-k plan statistics: [steps, passes, fused ops, unfused array kernels, measurements]
extern "C" int fs_debug_hbm_plan(fs_prog* p, int64_t* out) {
  if (!p || plan_hbm(p, p->dp.num_instrs, true)) return -1;
  const HbmPlan& PL = p->hplan;
  int64_t arr = 0, meas = 0;
  for (auto& st : PL.steps) { arr += st.kind == HbmStep::ARR; meas += st.kind == HbmStep::MEAS; }
  out[0] = (int64_t)PL.steps.size(); out[1] = (int64_t)PL.passes.size(); out[2] = (int64_t)PL.tileops.size();
  out[3] = arr; out[4] = meas;
  // microcode census: smem exchanges, register mixing ops, diagonal runs, code words
  int64_t sw = 0, mix = 0, dr = 0;
  for (auto& D : PL.passes)
    for (int pc = D.code_off; pc < D.code_off + D.ncode;) {
      const uint32_t w = PL.code[pc];
      const uint32_t k = w & 15u;
      if (k == fs::MC_DIAG) { dr++; pc += 8 + 2 * ((w >> 4) & 0xFF) + ((w >> 12) & 0xFF); continue; }
      const int m = (w >> 4) & 15;
      sw += m < 8;  // exchanges through shared memory
      mix += m >= 8;
      pc++;
    }
  out[5] = sw; out[6] = mix; out[7] = dr; out[8] = (int64_t)PL.code.size();
  return 0;
}

// live dimension (tile bits + base axes) of every fused pass, in execution order
extern "C" int64_t fs_debug_hbm_pass_bits(fs_prog* p, int32_t* out, int64_t max) {
  if (!p || plan_hbm(p, p->dp.num_instrs, true)) return -1;
  const HbmPlan& PL = p->hplan;
  int64_t n = 0;
  for (const HbmStep& st : PL.steps)
    if (st.kind == HbmStep::PASS) {
      if (n < max) out[n] = fs::kTileBits + PL.passes[st.pass].nbase;
      n++;
    }
  return n;
}

// per fused op: (pass, kind, la, lb, diag_run); returns the op count
extern "C" int64_t fs_debug_hbm_tileops(fs_prog* p, int32_t* out, int64_t max) {
  if (!p || plan_hbm(p, p->dp.num_instrs, true)) return -1;
  const HbmPlan& PL = p->hplan;
  int64_t n = 0;
  for (size_t ps = 0; ps < PL.passes.size(); ps++)
    for (int k = 0; k < PL.passes[ps].nops; k++, n++) {
      if (n >= max) continue;
      const fs::TileOp& o = PL.tileops[PL.passes[ps].op_off + k];
      int32_t* r = out + 5 * n;
      r[0] = (int32_t)ps; r[1] = o.kind; r[2] = o.la; r[3] = o.lb; r[4] = o.diag_run;
    }
  return n;
}

// kernel launches issued by this program so far (all engines, all kernels of this library)
extern "C" uint64_t fs_debug_launches(const fs_prog* p) { return p ? p->launches : 0; }

// enable (1) / disable (0) CUDA events around the dominant kernel's launches; resets the record
extern "C" int fs_debug_kernel_timer(fs_prog* p, int enable) {
  if (!p) return -1;
  std::lock_guard<std::mutex> g(p->mu);
  p->ktimer = enable != 0;
  p->kev_n = 0;
  return 0;
}

// total device time (ms) and count of the recorded dominant-kernel launches (synchronizes)
extern "C" int fs_debug_kernel_time(fs_prog* p, double* total_ms, int64_t* count) {
  if (!p) return -1;
  std::lock_guard<std::mutex> g(p->mu);
  double t = 0.0;
  for (size_t i = 0; i + 1 < p->kev_n; i += 2) {
    float ms = 0.f;
    if (cudaEventSynchronize(p->kev[i + 1]) != cudaSuccess) return -1;
    if (cudaEventElapsedTime(&ms, p->kev[i], p->kev[i + 1]) != cudaSuccess) return -1;
    t += ms;
  }
  *total_ms = t;
  *count = (int64_t)(p->kev_n / 2);
  return 0;
}

// per-launch device times (ms) of the recorded dominant-kernel launches; returns the count
extern "C" int64_t fs_debug_kernel_times(fs_prog* p, double* out, int64_t max) {
  if (!p) return -1;
  std::lock_guard<std::mutex> g(p->mu);
  int64_t n = 0;
  for (size_t i = 0; i + 1 < p->kev_n; i += 2, n++) {
    float ms = 0.f;
    if (cudaEventSynchronize(p->kev[i + 1]) != cudaSuccess) return -1;
    cudaEventElapsedTime(&ms, p->kev[i], p->kev[i + 1]);
    if (n < max) out[n] = ms;
  }
  return n;
}

extern "C" const char* fs_debug_jit_status(fs_prog* p) {
  static thread_local std::string s;
  if (!p) return "null";
  s = p->jit_state == 1 ? "ready compile_bytes=" + std::to_string(p->jit.cubin_bytes)
                        : (p->jit_state == 0 ? "not built" : "failed: " + p->jit_error);
  s += p->aff_state == 1 ? "; affine: ready threads=" + std::to_string(p->aff_threads)
                         : (p->aff_state == 0 ? "; affine: not built" : "; affine: n/a (" + p->aff_error + ")");
  s += p->seg_jit == 1 ? "; segments: ready kernels=" + std::to_string(p->seg_fn.size() - p->seg_lane.size()) + " lane=" + std::to_string(p->seg_lane.size())
                       : (p->seg_jit == 0 ? "; segments: not built" : "; segments: failed (" + p->seg_jit_err + ")");
  return s.c_str();
}

extern "C" int fs_program_engine(const fs_prog* p, uint32_t flags) {
  if (!p) return set_error(FS_ERR_ARG, "null program");
  if (wants_hbm(p, flags)) return 2;
  return wants_general(p, flags, nullptr, nullptr) ? 0 : 1;
}

namespace {

// events around the dominant kernel of an engine (bench.py: roofline of that kernel)
void kt_begin(fs_prog* p, cudaStream_t s) {
  if (!p->ktimer) return;
  while (p->kev.size() < p->kev_n + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) { p->ktimer = false; return; }
    p->kev.push_back(e);
  }
  cudaEventRecord(p->kev[p->kev_n], s);
}
void kt_end(fs_prog* p, cudaStream_t s) {
  if (!p->ktimer || p->kev.size() < p->kev_n + 2) return;
  cudaEventRecord(p->kev[p->kev_n + 1], s);
  p->kev_n += 2;
}

template <class K>
int occupancy_blocks(K kernel, int threads, size_t smem) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess) return 1;
  return std::max(nb, 1);
}


// ------------------------------------------------------------------ program-specialised kernel
int ensure_jit(fs_prog* p) {
  if (p->jit_state == 1) return FS_OK;
  if (p->jit_state == -1) return set_error(FS_ERR_ARG, p->jit_error);
  p->jit_state = -1;
  fsjit::FrameKernelSource K = fsjit::gen_frame_kernel(p->desc, p->h_instrs, p->h_gates, p->h_paulis, p->h_reclists,
                                                       p->h_record_out, p->h_bit_slot, p->h_plans,
                                                       p->h_case_pauli_off, p->h_site_case_off, p->h_site_prob);
  const size_t smem = (size_t)4 * (K.nslots + K.stage) * 32 * sizeof(uint32_t);
  if (smem > kSmemBudget) { p->jit_error = "frame too large for the specialised kernel"; return FS_ERR_ARG; }
  std::string err = fsjit::compile(K.src, fsjit::self_dir() + "/../csrc", p->jit);
  if (!err.empty()) { p->jit_error = err; return set_error(FS_ERR_ARG, err); }
  fsjit::Api& J = fsjit::api();
  if (J.cuFuncSetAttribute(p->jit.fn, 8 /* MAX_DYNAMIC_SHARED_SIZE_BYTES */, (int)smem) != 0) {
    p->jit_error = "cuFuncSetAttribute failed";
    return FS_ERR_ARG;
  }
  FS_CUDA_TRY(cudaMalloc(&p->d_pslot, sizeof(uint16_t) * K.pslot.size()));
  FS_CUDA_TRY(cudaMemcpy(p->d_pslot, K.pslot.data(), sizeof(uint16_t) * K.pslot.size(), cudaMemcpyHostToDevice));
  p->jit_nslots = K.nslots;
  p->jit_nblocks = K.nblocks;
  p->jit_stage = K.stage;
  FS_CUDA_TRY(cudaMalloc(&p->d_site_block, sizeof(int) * K.site_block.size()));
  FS_CUDA_TRY(cudaMemcpy(p->d_site_block, K.site_block.data(), sizeof(int) * K.site_block.size(), cudaMemcpyHostToDevice));
  p->jit_state = 1;
  return FS_OK;
}


// affine frame kernel (fs_affine.cuh) for frame-only programs, Philox free sampling
int ensure_aff(fs_prog* p) {
  if (p->aff_state == 1) return FS_OK;
  if (p->aff_state == -1) return FS_ERR_ARG;
  p->aff_state = -1;
  fsjit::AffineKernelSource K = fsjit::gen_affine_frame_kernel(
      p->desc, p->h_instrs, p->h_gates, p->h_paulis, p->h_reclists, p->h_record_out, p->h_bit_slot,
      p->h_case_pauli_off, p->h_site_case_off, p->h_site_prob, p->h_case_cum, kAffSmemBudget);
  if (!K.why.empty()) { p->aff_error = K.why; return FS_ERR_ARG; }
  std::string err = fsjit::compile(K.src, fsjit::self_dir() + "/../csrc", p->aff, "fs_aff_frame");
  if (!err.empty()) { p->aff_error = err; return set_error(FS_ERR_ARG, err); }
  fsjit::Api& J = fsjit::api();
  if (J.cuFuncSetAttribute(p->aff.fn, 8 /* MAX_DYNAMIC_SHARED_SIZE_BYTES */, (int)K.smem) != 0) {
    p->aff_error = "cuFuncSetAttribute failed";
    return FS_ERR_ARG;
  }
  FS_CUDA_TRY(cudaMalloc(&p->d_aff_tables, sizeof(uint32_t) * K.tables.size()));
  FS_CUDA_TRY(cudaMemcpy(p->d_aff_tables, K.tables.data(), sizeof(uint32_t) * K.tables.size(), cudaMemcpyHostToDevice));
  p->aff_threads = K.threads;
  p->aff_rows = K.nrows;
  p->aff_smem = K.smem;
  p->aff_state = 1;
  return FS_OK;
}

int launch_aff(fs_prog* p, fs::RunArgs& a, cudaStream_t stream) {
  fsjit::Api& J = fsjit::api();
  if (p->aff_occ == 0) {  // once per program: the launch path stays free of driver queries
    int occ = 1;
    J.cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->aff.fn, p->aff_threads, p->aff_smem);
    p->aff_occ = std::max(occ, 1);
  }
  const size_t groups = (a.W + 7) / 8, pairs = p->aff_threads / 64;  // one 8-word group per warp pair
  const size_t blocks = (groups + pairs - 1) / pairs;
  const size_t grid = std::min<size_t>(std::max<size_t>(blocks, 1), (size_t)p->num_sms * p->aff_occ);
  fs::DevProg dpv = p->dp;
  const uint32_t* tb = p->d_aff_tables;
  void* args[] = {&dpv, &a, &tb};
  kt_begin(p, stream);
  int r = J.cuLaunchKernel(p->aff.fn, (unsigned)grid, 1, 1, (unsigned)p->aff_threads, 1, 1, (unsigned)p->aff_smem,
                           stream, args, nullptr);
  kt_end(p, stream);
  p->launches++;
  if (r != 0) return set_error(FS_ERR_CUDA, "cuLaunchKernel(fs_aff_frame) failed: " + std::to_string(r));
  return FS_OK;
}


// one general-engine launch (array capacity 2^karr per lane; `units` = 32-shot groups)
int launch_general_kernel(fs_prog* p, fs::RunArgs& a, fs::SegArgs& S, bool seg, int karr, size_t units,
                          cudaStream_t stream) {
  const fs::DevProg& dp = p->dp;
  const bool splitmix = a.flags & FS_RNG_SPLITMIX;
  const int words_per_warp = (int)align_up(2 * dp.n + dp.num_slots + dp.O, 4);
  const size_t words_bytes = (size_t)fs::kGenWarps * words_per_warp * 4;
  const size_t arr_bytes_warp = ((size_t)32 << karr) * sizeof(double2);
  const bool arr_smem = words_bytes + 16 + fs::kGenWarps * arr_bytes_warp <= kSmemBudget;
  const size_t smem = words_bytes + (arr_smem ? 16 + fs::kGenWarps * arr_bytes_warp : 0);
  if (words_bytes > kSmemBudget) return set_error(FS_ERR_ARG, "program too large for the general engine");
  void (*kern)(fs::DevProg, fs::RunArgs, int, fs::SegArgs);
#define FS_PICK(SM, AS, SG) kern = fs::general_kernel<SM, AS, SG>
  if (seg) {
    if (splitmix) { if (arr_smem) FS_PICK(true, true, true); else FS_PICK(true, false, true); }
    else { if (arr_smem) FS_PICK(false, true, true); else FS_PICK(false, false, true); }
  } else {
    if (splitmix) { if (arr_smem) FS_PICK(true, true, false); else FS_PICK(true, false, false); }
    else { if (arr_smem) FS_PICK(false, true, false); else FS_PICK(false, false, false); }
  }
#undef FS_PICK
  FS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int threads = fs::kGenWarps * 32;
  const size_t blocks_needed = std::max<size_t>(1, (units + fs::kGenWarps - 1) / fs::kGenWarps);
  const int occ = occupancy_blocks(kern, threads, smem);
  size_t grid = std::min<size_t>(blocks_needed, (size_t)p->num_sms * occ);
  a.arr_log2 = karr;
  if (!arr_smem) {
    // HBM slab per resident warp; cap the footprint at ~48 GiB
    const size_t per_block = fs::kGenWarps * arr_bytes_warp;
    const size_t cap_blocks = std::max<size_t>(1, ((size_t)48 << 30) / per_block);
    grid = std::min(grid, cap_blocks);
    const size_t need = grid * per_block;
    if (need > p->scratch_bytes) {
      cudaFree(p->scratch);
      p->scratch = nullptr;
      p->scratch_bytes = 0;
      FS_CUDA_TRY(cudaMalloc(&p->scratch, need));
      p->scratch_bytes = need;
    }
    a.scratch = p->scratch;
  }
  kt_begin(p, stream);
  kern<<<(unsigned)grid, threads, smem, stream>>>(p->dp, a, words_per_warp, S);
  kt_end(p, stream);
  p->launches++;
  FS_CUDA_TRY(cudaGetLastError());
  return FS_OK;
}

// shot-per-warp (k <= 10) or shot-per-CTA launch for a segment with a large active array
// ------------------------------------------------------------------ specialised segment kernels
// The block engine's segments (warp- or CTA-per-shot) compiled to straight-line code (NVRTC):
// every array sweep becomes unrolled strips at constant offsets -- an element index is
// L(thread) | C(iteration) with both parts deposits of disjoint bit sets -- with the same
// per-thread order of partial sums as the interpreter (bit-identical results).  Scalar runs and
// the measurement decision call the shared BlockCtx members.
void gen_segment(std::ostringstream& o, const fs_prog* p, int b, int e, int karr, int G) {
  const int* IN = p->h_instrs.data();
  const int lg = G == 32 ? 5 : 8;
  o << "extern \"C\" __global__ void __launch_bounds__(" << (G == 32 ? 32 * fs::kBlockMaxGroups : 256) << ", "
    << (G == 32 ? 1 : 4) << ") fs_seg_" << b << "(DevProg P, RunArgs A, SegArgs S, int group_bytes) {\n"
    << "  block_run<false, " << G << ">(P, A, S, " << karr << ", group_bytes, [&](BlockCtx<false, " << G
    << ">& c) {\n    double2* __restrict__ am = c.amp;\n    const uint32_t tid = (uint32_t)c.tid;\n";
  // a strip loop over n items (constant trip count, compact code): `it` is the strip index,
  // `jj` = tid + G * it; items beyond n (n < G) are masked
  auto loop = [&](uint32_t nitems, const std::string& body) {
    const uint32_t nit = std::max<uint32_t>(1, nitems >> lg);
    const std::string guard = nitems < (uint32_t)G ? "if (tid < " + std::to_string(nitems) + "u) " : "";
    o << "      #pragma unroll 2\n      for (uint32_t it = 0; it < " << nit << "u; it++) " << guard << "{ const uint32_t jj = tid + (it << "
      << lg << "); " << body << " }\n";
  };
  for (int i = b; i < e;) {
    int j = std::min(p->h_next_array[i], e);
    if (j > i) {
      o << "    c.scalar_run(" << i << ", " << j << ");\n    if (!c.sh_alive) return;\n";
      i = j;
      continue;
    }
    const int* I = IN + (size_t)i * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]), flip = FS_FLIP(I[0]);
    const uint32_t size = 1u << I[6];
    if (op == FS_OP_ARRAY_GATE && p->h_fuse_at[i] >= 0) {  // a star group: frame matrix + one sweep
      const int32_t* Dg = p->h_fuse.data() + (size_t)8 * p->h_fuse_at[i];
      o << "    {  // " << i << " .. " << i + Dg[0] << "\n      c.frame_matrix(" << Dg[7] << ");\n      c.star_group("
        << (Dg[1] & 0xFF) << ", " << (uint32_t)Dg[2] << "u, " << (uint32_t)Dg[3] << "u, " << (Dg[4] & 3) << "u, "
        << ((Dg[4] & 4) ? "true" : "false") << ", " << ((Dg[4] & 8) ? "true" : "false") << ", " << (Dg[5] & 0xFFFF) << ", "
        << (Dg[5] >> 16) << ", " << Dg[6] << ", " << size << "u);\n    }\n";
      i += Dg[0];
      continue;
    }
    o << "    {  // " << i << "\n";
    switch (op) {
      case FS_OP_FRAME:
        o << "      c.frame_matrix(" << p->h_frame_mat_off[i] << ");\n";
        break;
      case FS_OP_ARRAY_GATE: {
        const int g = I[1], va = I[2], vb = I[3], a = I[4], bb = I[5];
        const uint32_t ia = 1u << a, ib = 1u << bb;
        if (g == FS_G_H)
          loop(size / 2, "const uint32_t i0 = ins0(jj, " + std::to_string(a) + "); const double2 lo = am[i0], hi = am[i0 + " +
                             std::to_string(ia) + "u]; am[i0] = cscale(cadd(lo, hi), kInvSqrt2); am[i0 + " + std::to_string(ia) +
                             "u] = cscale(csub(lo, hi), kInvSqrt2);");
        else if (g == FS_G_S || g == FS_G_SDAG)
          loop(size / 2, "const uint32_t i1 = ins0(jj, " + std::to_string(a) + ") + " + std::to_string(ia) +
                             "u; am[i1] = cmul(am[i1], make_double2(0.0, " + (g == FS_G_S ? "1.0" : "-1.0") + "));");
        else {
          const int lo = std::min(a, bb), hi = std::max(a, bb);
          const std::string id = "const uint32_t id = ins0(ins0(jj, " + std::to_string(lo) + "), " + std::to_string(hi) + ") + " +
                                 std::to_string(ia) + "u; ";
          if (g == FS_G_CX)
            loop(size / 4, id + "const double2 t0 = am[id]; am[id] = am[id + " + std::to_string(ib) + "u]; am[id + " +
                               std::to_string(ib) + "u] = t0;");
          else
            loop(size / 4, id + "const double2 v = am[id + " + std::to_string(ib) + "u]; am[id + " + std::to_string(ib) +
                               "u] = make_double2(-v.x, -v.y);");
        }
        o << "      c.gate_frame(" << g << ", " << va << ", " << vb << ");\n";
        break;
      }
      case FS_OP_EXPAND:
        o << "      double2 ph0, ph1;\n      c.parity_phases(" << I[1] << ", " << I[5] << ", 4, ph0, ph1);\n";
        loop(size, "const double2 v = am[jj]; am[jj] = cmul(v, ph0); am[jj + " + std::to_string(size) + "u] = cmul(v, ph1);");
        o << "      c.bar();\n";
        break;
      case FS_OP_ARRAY_ROT:
        o << "      double2 e0, e1;\n      c.parity_phases(" << I[1] << ", " << I[5] << ", 0, e0, e1);\n"
          << "      const int par = c.fx[" << I[1] << "] & 1;\n      const double2 ph0 = par ? e1 : e0, ph1 = par ? e0 : e1;\n";
        loop(size, "am[jj] = cmul(am[jj], ((jj >> " + std::to_string(I[2]) + ") & 1u) ? ph1 : ph0);");
        o << "      c.bar();\n";
        break;
      case FS_OP_MEAS_ACTIVE:
      case FS_OP_MEAS_COLLAPSE: {
        const bool collapse = op == FS_OP_MEAS_COLLAPSE;
        const int virt = I[1], a = I[2], rec = I[3];
        const uint32_t half = size >> 1, st = 1u << a;
        o << "      double2 u00 = make_double2(1, 0), u01 = make_double2(0, 0), u10 = make_double2(0, 0), u11 = make_double2(1, 0);\n";
        if (collapse) o << "      c.collapse_fparams(" << I[5] << ", u00, u01, u10, u11);\n";
        o << "      double s1 = 0.0, sa = 0.0;\n";
        loop(half, "const uint32_t i0 = ins0(jj, " + std::to_string(a) + "); const double2 a0 = am[i0], a1 = am[i0 + " + std::to_string(st) +
                       "u]; " + (collapse ? "s1 = __dadd_rn(s1, cnorm2(cadd(cmul(a0, u10), cmul(u11, a1)))); "
                                          : "s1 = __dadd_rn(s1, cnorm2(a1)); ") +
                       "sa = __dadd_rn(sa, __dadd_rn(cnorm2(a0), cnorm2(a1)));");
        o << "      c.reduce2(s1, sa);\n      c.meas_decide(" << i << ", " << (collapse ? "true" : "false") << ", " << virt << ", " << rec
          << ", " << flip << ", " << I[4] << ", s1, sa, u00, u01, u10, u11);\n      if (!c.sh_alive) return;\n"
          << "      c.branch = c.sh_branch;\n";
        if (collapse) {
          const std::string gd = half < (uint32_t)G ? "tid < " + std::to_string(half) + "u" : "true";
          o << "      const double2 k0 = c.sh_k0, k1 = c.sh_k1;\n"
            << "      for (uint32_t b0 = 0; b0 < " << half << "u; b0 += " << G << "u) {\n"
            << "        const uint32_t jj = b0 + tid;\n        double2 val = make_double2(0.0, 0.0);\n"
            << "        if (" << gd << ") { const uint32_t i0 = ins0(jj, " << a << "); val = cadd(cmul(k0, am[i0]), cmul(k1, am[i0 + "
            << st << "u])); }\n        c.bar();\n        if (" << gd << ") am[jj] = val;\n        c.bar();\n      }\n";
        } else {
          o << "      const double s = c.sh_k0.x;\n      const uint32_t dead = 1u - (uint32_t)c.branch;\n";
          loop(size, "if (((jj >> " + std::to_string(a) + ") & 1u) == dead) am[jj] = make_double2(0.0, 0.0); else if (c.renorm) am[jj] = cscale(am[jj], s);");
        }
        o << "      c.bar();\n";
        break;
      }
      case FS_OP_RETIRE:
        o << "      c.retire(" << I[1] << ", " << I[2] << ", " << size << "u);\n";
        break;
      default:
        break;
    }
    o << "    }\n";
    i++;
  }
  o << "  });\n}\n";
}

// Warp-per-shot segments fully specialised (fs_wseg.cuh): scalar instructions included, the frame
// bit-packed in registers.  Needs 2n <= 128 (frame matrices, case masks), <= 32 slots / observables.
// threads of a CTA of G-thread shots: 16 warp shots, 15 two-warp shots (named barriers 1..15), one
// CTA-wide shot
int wseg_groups(int G) { return G == 32 ? fs::kBlockMaxGroups : (G == 256 ? 1 : 15); }
int wseg_threads(int G) { return G * wseg_groups(G); }

bool wseg_supported(const fs_prog* p) {
  return 2 * p->dp.n <= 128 && p->dp.num_slots <= 32 && p->dp.O <= 32 && p->dp.case_mask != nullptr;
}

void gen_segment_w(std::ostringstream& o, const fs_prog* p, int b, int e, int karr, int G) {
  const int* IN = p->h_instrs.data();
  const int n = p->dp.n, R = p->dp.R;
  auto C = [&](int off) {
    return "make_double2(" + fsjit::hexd(p->h_fparams[off]) + ", " + fsjit::hexd(p->h_fparams[off + 1]) + ")";
  };
  auto slot_of = [&](int bit) { return p->h_bit_slot[bit]; };
  // mask words of a Pauli list
  auto mask_of = [&](int off, int cnt, uint32_t m[4]) {
    m[0] = m[1] = m[2] = m[3] = 0u;
    for (int j = off; j < off + cnt; j++) {
      const uint32_t en = p->h_paulis[j];
      const int bit = FS_PAULI_Z(en) ? n + (int)FS_PAULI_Q(en) : (int)FS_PAULI_Q(en);
      m[bit >> 5] ^= 1u << (bit & 31);
    }
  };
  auto frame_gate = [&](int g, int va, int vb) {
    switch (g) {
      case FS_G_S: case FS_G_SDAG: o << "    c.g_s(" << va << ", " << n + va << ");\n"; break;
      case FS_G_H: o << "    c.g_h(" << va << ", " << n + va << ");\n"; break;
      case FS_G_CX: o << "    c.g_cx(" << va << ", " << n + va << ", " << vb << ", " << n + vb << ");\n"; break;
      case FS_G_CZ: o << "    c.g_cz(" << va << ", " << n + va << ", " << vb << ", " << n + vb << ");\n"; break;
      case FS_G_SWAP: o << "    c.g_swap(" << va << ", " << n + va << ", " << vb << ", " << n + vb << ");\n"; break;
      default: break;
    }
  };
  // the frame side of instructions [i0, i1) gate by gate: register instructions at constant bit
  // positions (the GF(2) frame matrices of the interpreter cost a row load per frame bit: measured
  // 43.1 vs 41.5 ms per 16.8M shots of config 4)
  auto frame_updates = [&](int i0, int i1) {
    for (int i = i0; i < i1; i++) {
      const int* I = IN + (size_t)i * FS_INS_WORDS;
      const int op = FS_OPCODE(I[0]);
      if (op == FS_OP_FRAME) {
        for (int j = 0; j < I[2]; j++) {
          const uint32_t g = p->h_gates[I[1] + j];
          frame_gate(FS_GATE_G(g), FS_GATE_A(g), FS_GATE_B(g));
        }
      } else if (op == FS_OP_ARRAY_GATE) {
        frame_gate(I[1], I[2], I[3]);
      }
    }
  };
  o << "extern \"C\" __global__ void __launch_bounds__(" << wseg_threads(G) << ", " << (G == 256 ? (karr <= 11 ? 4 : 3) : 1) << ") fs_seg_" << b
    << "(DevProg P, RunArgs A, SegArgs S, int group_bytes) {\n  wseg_run<" << G << ", " << karr << ">(P, A, S, group_bytes, [&](WCtxT<" << G
    << ">& c) {\n";
  for (int i = b; i < e;) {
    const int* I = IN + (size_t)i * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]), flip = FS_FLIP(I[0]);
    const uint32_t size = 1u << I[6];
    o << "    // " << i << "\n";
    if (op == FS_OP_ARRAY_GATE && p->h_fuse_at[i] >= 0) {
      const int32_t* Dg = p->h_fuse.data() + (size_t)8 * p->h_fuse_at[i];
      const bool hasAR = (Dg[4] & 8) != 0;
      frame_updates(i, i + Dg[0]);
      o << "    {\n";
      if (hasAR) {
        const int virt = Dg[5] & 0xFFFF, fp = Dg[6];
        o << "      const uint32_t par = c.fbit(" << virt << ");\n      const double2 e0 = " << C(fp) << ", e1 = " << C(fp + 2)
          << ";\n      const double2 ph0 = par ? e1 : e0, ph1 = par ? e0 : e1;\n";
      } else {
        o << "      const double2 ph0 = make_double2(1.0, 0.0), ph1 = ph0;\n";
      }
      o << "      c.star<" << ((Dg[4] & 1) ? "true" : "false") << ">(" << (Dg[1] & 0xFF) << ", " << (uint32_t)Dg[2] << "u, "
        << (uint32_t)Dg[3] << "u, " << (Dg[4] & 3) << "u, " << ((Dg[4] & 4) ? "true" : "false") << ", "
        << (hasAR ? "true" : "false") << ", " << (Dg[5] >> 16) << ", ph0, ph1, " << size << "u);\n    }\n";
      i += Dg[0];
      continue;
    }
    switch (op) {
      case FS_OP_FRAME:
        frame_updates(i, i + 1);
        break;
      case FS_OP_ARRAY_GATE:
        o << "    c.gate(" << I[1] << ", " << I[4] << ", " << I[5] << ", " << size << "u);\n";
        frame_gate(I[1], I[2], I[3]);
        break;
      case FS_OP_EXPAND:
        o << "    { const uint32_t par = c.fbit(" << I[1] << "); c.expand(" << size << "u, par ? " << C(I[5] + 4) << " : " << C(I[5])
          << ", par ? " << C(I[5] + 6) << " : " << C(I[5] + 2) << "); }\n";
        break;
      case FS_OP_ARRAY_ROT:
        o << "    { const uint32_t par = c.fbit(" << I[1] << "); const double2 e0 = " << C(I[5]) << ", e1 = " << C(I[5] + 2)
          << "; c.array_rot(" << I[2] << ", " << size << "u, par ? e1 : e0, par ? e0 : e1); }\n";
        break;
      case FS_OP_MEAS_DSTATIC:
        o << "    c.meas_dstatic(" << I[1] << ", " << flip << ", " << p->h_record_out[I[3]] << ", " << slot_of(I[3]) << ");\n";
        break;
      case FS_OP_MEAS_DRANDOM:
        o << "    c.meas_drandom(" << I[1] << ", " << n + I[1] << ", " << I[2] << ", " << flip << ", " << p->h_record_out[I[3]] << ", "
          << slot_of(I[3]) << ");\n";
        break;
      case FS_OP_MEAS_ACTIVE:
      case FS_OP_MEAS_COLLAPSE: {
        const bool collapse = op == FS_OP_MEAS_COLLAPSE;
        if (collapse) {
          const int po = I[4] >> 8, pc = I[4] & 0xFF;
          for (int j = 0; j < pc; j++) {
            const uint32_t g = p->h_gates[po + j];
            frame_gate(FS_GATE_G(g), FS_GATE_A(g), FS_GATE_B(g));
          }
        }
        o << "    if (!c.measure<" << (collapse ? "true" : "false") << ">(" << i << ", " << I[1] << ", " << I[2] << ", " << flip << ", "
          << p->h_record_out[I[3]] << ", " << slot_of(I[3]) << ", " << size << "u, ";
        if (collapse) o << C(I[5]) << ", " << C(I[5] + 2) << ", " << C(I[5] + 4) << ", " << C(I[5] + 6);
        else o << "make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0)";
        o << ")) return;\n";
        break;
      }
      case FS_OP_RETIRE:
        o << "    c.retire(" << I[1] << ", " << I[2] << ", " << size << "u);\n";
        break;
      case FS_OP_COND_FRAME: {
        uint32_t m[4];
        mask_of(I[1], I[2], m);
        o << "    if ((c.slots >> " << slot_of(I[3]) << ") & 1u) c.xor_mask(" << m[0] << "u, " << m[1] << "u, " << m[2] << "u, " << m[3]
          << "u);\n";
        break;
      }
      case FS_OP_NOISE:
        o << "    c.noise(" << I[2] << ");\n";
        break;
      case FS_OP_DETECTOR:
      case FS_OP_OBSERVABLE: {
        o << "    { const uint32_t v = (0u";
        for (int j = 0; j < I[3]; j++) o << " ^ (c.slots >> " << slot_of(p->h_reclists[I[2] + j]) << ")";
        o << ") & 1u; ";
        if (op == FS_OP_DETECTOR) o << "c.detector(v, " << I[1] << ", " << slot_of(R + I[1]) << "); }\n";
        else o << "c.obs ^= v << " << I[1] << "; }\n";
        break;
      }
      case FS_OP_POSTSELECT: {
        const int bid = I[1] == 0 ? R + I[2] : I[2];
        o << "    if (((c.slots >> " << slot_of(bid) << ") & 1u) != " << I[3] << "u) { c.alive = 0; return; }\n";
        break;
      }
      default:
        break;  // GammaRot: the global phase is not an output of free sampling
    }
    i++;
  }
  o << "  });\n}\n";
}

// Lane-per-shot segments fully specialised (fs_lseg.cuh): every lane runs one shot with its frame
// packed in registers and its array in a per-thread array.  Same limits as the warp-per-shot form.
constexpr int kLsegMaxK = 8;  // 2^8 amplitudes = 4 KiB of thread-local memory per shot

void gen_segment_l(std::ostringstream& o, const fs_prog* p, int b, int e, int karr, int k_in, int k_out) {
  const int* IN = p->h_instrs.data();
  const int n = p->dp.n, R = p->dp.R;
  auto C = [&](int off) {
    return "make_double2(" + fsjit::hexd(p->h_fparams[off]) + ", " + fsjit::hexd(p->h_fparams[off + 1]) + ")";
  };
  auto slot_of = [&](int bit) { return p->h_bit_slot[bit]; };
  auto mask_of = [&](int off, int cnt, uint32_t m[4]) {
    m[0] = m[1] = m[2] = m[3] = 0u;
    for (int j = off; j < off + cnt; j++) {
      const uint32_t en = p->h_paulis[j];
      const int bit = FS_PAULI_Z(en) ? n + (int)FS_PAULI_Q(en) : (int)FS_PAULI_Q(en);
      m[bit >> 5] ^= 1u << (bit & 31);
    }
  };
  auto frame_gate = [&](int g, int va, int vb) {
    switch (g) {
      case FS_G_S: case FS_G_SDAG: o << "    c.g_s(" << va << ", " << n + va << ");\n"; break;
      case FS_G_H: o << "    c.g_h(" << va << ", " << n + va << ");\n"; break;
      case FS_G_CX: o << "    c.g_cx(" << va << ", " << n + va << ", " << vb << ", " << n + vb << ");\n"; break;
      case FS_G_CZ: o << "    c.g_cz(" << va << ", " << n + va << ", " << vb << ", " << n + vb << ");\n"; break;
      case FS_G_SWAP: o << "    c.g_swap(" << va << ", " << n + va << ", " << vb << ", " << n + vb << ");\n"; break;
      default: break;
    }
  };
  // Expands after the last array-reading instruction are deferred to the save (fs_lseg.cuh)
  int lazy_from = b;
  for (int i = b; i < e; i++) {
    const int op = FS_OPCODE(IN[(size_t)i * FS_INS_WORDS]);
    if (op == FS_OP_ARRAY_GATE || op == FS_OP_ARRAY_ROT || op == FS_OP_MEAS_ACTIVE || op == FS_OP_MEAS_COLLAPSE || op == FS_OP_RETIRE)
      lazy_from = i + 1;
  }
  int nlazy = 0, karr_eff = k_in;
  for (int i = b; i < e; i++) {
    const int op = FS_OPCODE(IN[(size_t)i * FS_INS_WORDS]);
    if (i >= lazy_from && op == FS_OP_EXPAND) nlazy++;
    else if (i < lazy_from) karr_eff = std::max(karr_eff, p->h_sched[i]);
  }
  if (nlazy > 6) {  // keep the pending phase pairs few: the earliest Expands run eagerly
    int skip = nlazy - 6;
    for (int i = lazy_from; i < e && skip > 0; i++)
      if (FS_OPCODE(IN[(size_t)i * FS_INS_WORDS]) == FS_OP_EXPAND) { lazy_from = i + 1; karr_eff = std::max(karr_eff, p->h_sched[i]); skip--; nlazy--; }
  }
  (void)karr;
  o << "extern \"C\" __global__ void __launch_bounds__(128) fs_seg_" << b
    << "(DevProg P, RunArgs A, SegArgs S, int group_bytes) {\n  lseg_run<" << karr_eff << ", " << k_in << ", " << k_out << ", " << nlazy
    << ">(P, A, S, [&](LCtx<" << karr_eff << ", " << nlazy << ">& c) {\n";
  int lz = 0;
  for (int i = b; i < e; i++) {
    const int* I = IN + (size_t)i * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]), flip = FS_FLIP(I[0]);
    o << "    // " << i << "\n";
    switch (op) {
      case FS_OP_FRAME:
        for (int j = 0; j < I[2]; j++) {
          const uint32_t g = p->h_gates[I[1] + j];
          frame_gate(FS_GATE_G(g), FS_GATE_A(g), FS_GATE_B(g));
        }
        break;
      case FS_OP_ARRAY_GATE:
        o << "    c.gate<" << I[1] << ", " << I[4] << ", " << (I[5] < 0 ? 0 : I[5]) << ", " << I[6] << ">();\n";
        frame_gate(I[1], I[2], I[3]);
        break;
      case FS_OP_EXPAND:
        if (i >= lazy_from) {
          o << "    { const uint32_t par = c.fbit(" << I[1] << "); c.lz0[" << lz << "] = par ? " << C(I[5] + 4) << " : " << C(I[5])
            << "; c.lz1[" << lz << "] = par ? " << C(I[5] + 6) << " : " << C(I[5] + 2) << "; }\n";
          lz++;
          break;
        }
        o << "    { const uint32_t par = c.fbit(" << I[1] << "); c.expand<" << I[6] << ">(par ? " << C(I[5] + 4) << " : " << C(I[5])
          << ", par ? " << C(I[5] + 6) << " : " << C(I[5] + 2) << "); }\n";
        break;
      case FS_OP_ARRAY_ROT:
        o << "    { const uint32_t par = c.fbit(" << I[1] << "); const double2 e0 = " << C(I[5]) << ", e1 = " << C(I[5] + 2)
          << "; c.array_rot<" << I[2] << ", " << I[6] << ">(par ? e1 : e0, par ? e0 : e1); }\n";
        break;
      case FS_OP_MEAS_DSTATIC:
        o << "    c.meas_dstatic(" << I[1] << ", " << flip << ", " << p->h_record_out[I[3]] << ", " << slot_of(I[3]) << ");\n";
        break;
      case FS_OP_MEAS_DRANDOM:
        o << "    c.meas_drandom(" << I[1] << ", " << n + I[1] << ", " << I[2] << ", " << flip << ", " << p->h_record_out[I[3]] << ", "
          << slot_of(I[3]) << ");\n";
        break;
      case FS_OP_MEAS_ACTIVE:
      case FS_OP_MEAS_COLLAPSE: {
        const bool collapse = op == FS_OP_MEAS_COLLAPSE;
        if (collapse) {
          const int po = I[4] >> 8, pc = I[4] & 0xFF;
          for (int j = 0; j < pc; j++) {
            const uint32_t g = p->h_gates[po + j];
            frame_gate(FS_GATE_G(g), FS_GATE_A(g), FS_GATE_B(g));
          }
        }
        o << "    if (!c.measure<" << (collapse ? "true" : "false") << ", " << I[2] << ", " << I[6] << ">(" << i << ", " << I[1] << ", "
          << flip << ", " << p->h_record_out[I[3]] << ", " << slot_of(I[3]) << ", ";
        if (collapse) o << C(I[5]) << ", " << C(I[5] + 2) << ", " << C(I[5] + 4) << ", " << C(I[5] + 6);
        else o << "make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0)";
        o << ")) return;\n";
        break;
      }
      case FS_OP_RETIRE:
        o << "    c.retire<" << I[2] << ", " << I[6] << ">(" << I[1] << ");\n";
        break;
      case FS_OP_COND_FRAME: {
        uint32_t m[4];
        mask_of(I[1], I[2], m);
        o << "    if ((c.slots >> " << slot_of(I[3]) << ") & 1u) c.xor_mask(" << m[0] << "u, " << m[1] << "u, " << m[2] << "u, " << m[3]
          << "u);\n";
        break;
      }
      case FS_OP_NOISE:
        o << "    c.noise(" << I[2] << ");\n";
        break;
      case FS_OP_DETECTOR:
      case FS_OP_OBSERVABLE: {
        o << "    { const uint32_t v = (0u";
        for (int j = 0; j < I[3]; j++) o << " ^ (c.slots >> " << slot_of(p->h_reclists[I[2] + j]) << ")";
        o << ") & 1u; ";
        if (op == FS_OP_DETECTOR) o << "c.detector(v, " << I[1] << ", " << slot_of(R + I[1]) << "); }\n";
        else o << "c.obs ^= v << " << I[1] << "; }\n";
        break;
      }
      case FS_OP_POSTSELECT: {
        const int bid = I[1] == 0 ? R + I[2] : I[2];
        o << "    if (((c.slots >> " << slot_of(bid) << ") & 1u) != " << I[3] << "u) { c.alive = 0; return; }\n";
        break;
      }
      default:
        break;  // GammaRot: the global phase is not an output of free sampling
    }
  }
  o << "  });\n}\n";
}

// every block-engine segment of the program (Philox stream) in one NVRTC module
int ensure_seg_jit(fs_prog* p, const std::vector<int>& bounds, const std::vector<int>& karrs, int block_k) {
  if (p->seg_jit == 1) return FS_OK;
  if (p->seg_jit == -1) return FS_ERR_ARG;
  p->seg_jit = -1;
  std::ostringstream o;
  o << "#include \"fs_lseg.cuh\"\nusing namespace fs;\n";
  std::vector<int> begins;
  const int* sched = p->h_sched.data();
  // One kernel per PostSelect segment.  (Measured and not adopted: runs of consecutive warp- or CTA-
  // per-shot segments as ONE kernel, a shot staying in shared memory across its PostSelects -- 15 %
  // fewer instructions and no survivor-store round trips, but 77 vs 41.6 ms per 16.8M shots of
  // config 4: the warps of a CTA then sit in different segments' straight-line code and stall on
  // instruction fetch.)
  const bool packed = wseg_supported(p) && !p->env.block_no_wjit;
  const std::vector<int>& fb = bounds;
  const std::vector<int>& fk = karrs;
  for (size_t s = 0; s + 1 < fb.size(); s++) {
    const int karr = fk[s];
    if (karr < block_k) {
      // lane-per-shot segments: fully specialised (fs_lseg.cuh) while the array fits thread-local
      // memory; the interpreter otherwise
      if (karr > kLsegMaxK || !wseg_supported(p) || p->env.seg_no_ljit) continue;
      gen_segment_l(o, p, fb[s], fb[s + 1], karr, fb[s] > 0 ? sched[fb[s] - 1] : 0, sched[fb[s + 1] - 1]);
      p->seg_lane.insert(fb[s]);
    } else if (packed) {
      // warp-per-shot (k <= 10) and CTA-per-shot segments fully specialised, packed frame in
      // registers (fs_wseg.cuh); two warps per shot measured no faster than one at k = 9-10
      const int G = karr <= 10 ? 32 : 256;
      gen_segment_w(o, p, fb[s], fb[s + 1], karr, G);
      p->seg_G[fb[s]] = G;
    } else {
      // programs beyond the packed frame (2n > 128, > 32 slots) or FS_BLOCK_NO_WJIT: CTA-per-shot
      // segments as specialised sweeps around the shared scalar VM (measured 1.2-1.8x faster than
      // interpreted); warp-per-shot ones in that form ran ~2x slower than interpreted (instruction-
      // fetch stalls) and keep the interpreter
      if (karr <= 10) continue;
      gen_segment(o, p, fb[s], fb[s + 1], karr, 256);
    }
    begins.push_back(fb[s]);
  }
  if (begins.empty()) { p->seg_jit = 1; return FS_OK; }
  static std::mutex mu;  // modules belong to a context: key (current context, source)
  static std::map<std::pair<fsjit::CUcontext, std::string>, fsjit::CUmodule> cache;
  std::lock_guard<std::mutex> g(mu);
  const std::string src = o.str();
  if (!fsjit::api().ok) { p->seg_jit_err = fsjit::api().why; return FS_ERR_ARG; }
  fsjit::CUcontext ctx = nullptr;
  fsjit::api().cuCtxGetCurrent(&ctx);
  const auto key = std::make_pair(ctx, src);
  fsjit::CUmodule mod = nullptr;
  auto it = cache.find(key);
  if (it != cache.end()) {
    mod = it->second;
  } else {
    fsjit::Compiled c;
    std::string err = fsjit::compile(src, fsjit::self_dir() + "/../csrc", c, ("fs_seg_" + std::to_string(begins[0])).c_str());
    if (!err.empty()) { p->seg_jit_err = err; return FS_ERR_ARG; }
    mod = c.mod;
    cache[key] = mod;
  }
  for (int b : begins) {
    fsjit::CUfunction f = nullptr;
    if (fsjit::api().cuModuleGetFunction(&f, mod, ("fs_seg_" + std::to_string(b)).c_str()) != 0) {
      p->seg_jit_err = "missing segment kernel";
      return FS_ERR_ARG;
    }
    p->seg_fn[b] = f;
  }
  p->seg_jit = 1;
  return FS_OK;
}

int launch_block_kernel(fs_prog* p, fs::RunArgs& a, fs::SegArgs& S, int karr, cudaStream_t stream) {
  const fs::DevProg& dp = p->dp;
  // per shot: the array, then the interpreter's frame words / the packed-frame kernels' scratch
  const size_t group_bytes = align_up(((size_t)16 << karr) + std::max<size_t>(256, (size_t)4 * (2 * dp.n + dp.num_slots + dp.O + 4)), 16);
  if (group_bytes > kSmemBudget) return set_error(FS_ERR_ARG, "active array too large for the block engine");
  const bool sm = a.flags & FS_RNG_SPLITMIX;
  const bool trace = a.fault_modes || a.forced || a.t_fx || a.t_gamma || a.t_amps || a.t_draws || a.t_rec || a.ncp;
  auto fit = p->seg_fn.find(S.seg_begin);
  const bool jit = !sm && !trace && p->seg_jit == 1 && fit != p->seg_fn.end() && !p->env.block_no_jit;
  const bool warp_mode = karr <= 10;
  // threads per shot: the packed-frame kernels carry their own, else a warp (k <= 10) or a CTA
  auto git = p->seg_G.find(S.seg_begin);
  const int G = jit && git != p->seg_G.end() ? git->second : (warp_mode ? 32 : 256);
  // as many shots per CTA as fit next to the static shared arrays (a k = 10 shot is ~17 KB)
  const size_t dyn_budget = 220 * 1024;
  const int ngroups = G == 256 ? 1 : (int)std::max<size_t>(1, std::min<size_t>(wseg_groups(G), dyn_budget / group_bytes));
  const int nt = G * ngroups;
  const size_t smem = group_bytes * ngroups;
  void (*kern)(fs::DevProg, fs::RunArgs, fs::SegArgs, int, int);
  if (warp_mode) kern = sm ? fs::block_kernel<true, 32> : fs::block_kernel<false, 32>;
  else kern = sm ? fs::block_kernel<true, 256> : fs::block_kernel<false, 256>;
  const size_t blocks_needed = (S.n_in + ngroups - 1) / ngroups;
  if (jit) {  // specialised kernel
    fsjit::Api& J = fsjit::api();
    if (J.cuFuncSetAttribute(fit->second, 8, (int)smem) != 0) return set_error(FS_ERR_CUDA, "cuFuncSetAttribute(fs_seg)");
    int occ = 0;
    auto oit = p->seg_occ.find(S.seg_begin);  // threads and shared memory are fixed per segment
    if (oit != p->seg_occ.end()) occ = oit->second;
    else {
      if (J.cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fit->second, nt, smem) != 0 || occ < 1) occ = 1;
      p->seg_occ[S.seg_begin] = occ;
    }
    const size_t grid = std::max<size_t>(1, std::min<size_t>(blocks_needed, (size_t)p->num_sms * occ));
    fs::DevProg dpv = dp;
    fs::RunArgs av = a;
    fs::SegArgs sv = S;
    int gb = (int)group_bytes;
    void* args[] = {&dpv, &av, &sv, &gb};
    kt_begin(p, stream);
    const int r = J.cuLaunchKernel(fit->second, (unsigned)grid, 1, 1, nt, 1, 1, (unsigned)smem, stream, args, nullptr);
    kt_end(p, stream);
    p->launches++;
    if (r != 0) return set_error(FS_ERR_CUDA, "cuLaunchKernel(fs_seg) failed: " + std::to_string(r));
    return FS_OK;
  }
  FS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int occ = occupancy_blocks(kern, nt, smem);
  const size_t grid = std::max<size_t>(1, std::min<size_t>(blocks_needed, (size_t)p->num_sms * occ));
  kt_begin(p, stream);
  kern<<<(unsigned)grid, nt, smem, stream>>>(dp, a, S, karr, (int)group_bytes);
  kt_end(p, stream);
  p->launches++;
  FS_CUDA_TRY(cudaGetLastError());
  return FS_OK;
}

// lane-per-shot specialised segment (fs_lseg.cuh): Philox free sampling only
bool lseg_ready(const fs_prog* p, const fs::RunArgs& a, const fs::SegArgs& S) {
  const bool trace = a.fault_modes || a.forced || a.t_fx || a.t_gamma || a.t_amps || a.t_draws || a.t_rec || a.ncp;
  return !(a.flags & FS_RNG_SPLITMIX) && !trace && p->seg_jit == 1 && !p->env.block_no_jit &&
         p->seg_lane.count(S.seg_begin) && p->seg_fn.count(S.seg_begin);
}

int launch_lane_segment(fs_prog* p, fs::RunArgs& a, fs::SegArgs& S, cudaStream_t stream) {
  fsjit::Api& J = fsjit::api();
  fsjit::CUfunction fn = p->seg_fn[S.seg_begin];
  const int nt = 128;
  int occ = 0;
  auto oit = p->seg_occ.find(S.seg_begin);
  if (oit != p->seg_occ.end()) occ = oit->second;
  else {
    if (J.cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nt, 0) != 0 || occ < 1) occ = 1;
    p->seg_occ[S.seg_begin] = occ;
  }
  const size_t blocks_needed = ((size_t)S.n_in + nt - 1) / nt;
  const size_t grid = std::max<size_t>(1, std::min<size_t>(blocks_needed, (size_t)p->num_sms * occ));
  fs::DevProg dpv = p->dp;
  fs::RunArgs av = a;
  fs::SegArgs sv = S;
  int gb = 0;
  void* args[] = {&dpv, &av, &sv, &gb};
  kt_begin(p, stream);
  const int r = J.cuLaunchKernel(fn, (unsigned)grid, 1, 1, nt, 1, 1, 0, stream, args, nullptr);
  kt_end(p, stream);
  p->launches++;
  if (r != 0) return set_error(FS_ERR_CUDA, "cuLaunchKernel(fs_seg, lane) failed: " + std::to_string(r));
  return FS_OK;
}

// state store carve-out for `slots` survivors with arrays of 2^k
size_t store_bytes(const fs::DevProg& dp, const fs::SegArgs& S, size_t slots, int k) {
  const size_t sl = align_up(slots, 32);
  return align_up(sl * 4 * (S.nfw + S.nsw + S.now + 2 + 6), 256) + align_up(sl * 24, 256) +
         align_up(sl * 16 * ((size_t)1 << k), 256) + 4096;
}

fs::StateStore carve_store(void* base, const fs::SegArgs& S, size_t slots, int k) {
  Stage st;
  st.base = static_cast<unsigned char*>(base);
  const size_t sl = align_up(slots, 32);
  fs::StateStore o{};
  o.frame = st.take<uint32_t>(sl * S.nfw + 1);
  o.slotbits = st.take<uint32_t>(sl * S.nsw + 1);
  o.obsbits = st.take<uint32_t>(sl * S.now + 1);
  o.smcount = st.take<uint32_t>(sl);
  o.shot = st.take<uint32_t>(sl);
  o.gen_i = st.take<uint32_t>(sl * 6);
  o.gen_c = st.take<double>(sl);
  o.gamma = st.take<double2>(sl);
  o.amps = st.take<double2>(sl * ((size_t)1 << k));
  return o;
}

// Segmented general engine for programs with PostSelect (config 4): cut after every
// PostSelect, run each segment over the surviving shots only, compact survivors in between.
int launch_segmented(fs_prog* p, fs::RunArgs& a, cudaStream_t stream) {
  const fs::DevProg& dp = p->dp;
  const int* I = p->h_instrs.data();
  const int* sched = p->h_sched.data();
  std::vector<int> bounds{0};
  for (int i = 0; i < dp.num_instrs; i++)
    if (FS_OPCODE(I[(size_t)i * FS_INS_WORDS]) == FS_OP_POSTSELECT && i + 1 < dp.num_instrs) bounds.push_back(i + 1);
  bounds.push_back(dp.num_instrs);
  // outputs are OR-ed bit by bit once shots are compacted
  const size_t W = a.W;
  if (dp.U) FS_CUDA_TRY(cudaMemsetAsync(a.meas, 0, 4 * dp.U * W, stream));
  if (dp.D) FS_CUDA_TRY(cudaMemsetAsync(a.det, 0, 4 * dp.D * W, stream));
  if (dp.O) FS_CUDA_TRY(cudaMemsetAsync(a.obs, 0, 4 * dp.O * W, stream));
  FS_CUDA_TRY(cudaMemsetAsync(a.accepted, 0, 4 * W, stream));
  FS_CUDA_TRY(cudaMemsetAsync(a.error, 0, 4 * W, stream));
  a.prezeroed = 1;
  fs::SegArgs S{};
  S.nfw = (2 * dp.n + 31) / 32;
  S.nsw = (dp.num_slots + 31) / 32;
  S.now = (dp.O + 31) / 32;
  // star groups run fused unless a checkpoint asks for the state inside one
  S.fuse = 1;
  if (a.ncp)
    for (int c : p->cp_list)
      for (int i = 0; i < dp.num_instrs; i++)
        if (p->h_fuse_at[i] >= 0 && c > i && c < i + p->h_fuse[(size_t)8 * p->h_fuse_at[i]]) S.fuse = 0;
  // shots per pass over the segments: 2^23 measured 2 % faster than 2^22 on config 4 (the deep
  // segments' launches carry more shots), 2^24 the same; the k = 10 survivor store is ~9 GB
  const uint64_t chunk = (uint64_t)1 << 23;
  if (!p->d_counts) FS_CUDA_TRY(cudaMalloc(&p->d_counts, 64));
  uint32_t* d_nout = reinterpret_cast<uint32_t*>(p->d_counts);
  p->seg_counts.clear();
  int block_k = kBlockK;
  if (p->env.block_k) block_k = p->env.block_k;  // experiments
  if (!(a.flags & FS_RNG_SPLITMIX) && !p->env.block_no_jit && p->seg_jit == 0) {
    std::vector<int> karrs;
    for (int sgi = 0; sgi + 1 < (int)bounds.size(); sgi++) {
      int kk = bounds[sgi] > 0 ? sched[bounds[sgi] - 1] : 0;
      for (int i = bounds[sgi]; i < bounds[sgi + 1]; i++) kk = std::max(kk, sched[i]);
      karrs.push_back(kk);
    }
    ensure_seg_jit(p, bounds, karrs, block_k);  // failure leaves the interpreter in place
  }
  const int nseg = (int)bounds.size() - 1;
  for (uint64_t c0 = 0; c0 < a.nshots; c0 += chunk) {
    uint32_t n_in = (uint32_t)std::min<uint64_t>(chunk, a.nshots - c0);
    p->seg_counts.push_back(n_in);
    int cur = 0;  // which pool holds the input store
    for (int sgi = 0; sgi < nseg; sgi++) {
      const int b = bounds[sgi], e = bounds[sgi + 1];
      S.seg_begin = b;
      S.seg_end = e;
      S.first = sgi == 0;
      S.last = sgi == nseg - 1;
      S.n_in = n_in;
      S.chunk0 = c0;
      S.k_in = b > 0 ? sched[b - 1] : 0;
      S.k_out = sched[e - 1];
      int karr = S.k_in;
      for (int i = b; i < e; i++) karr = std::max(karr, sched[i]);
      // engine of the NEXT segment decides the survivor store layout
      int karr_next = 0;
      if (!S.last) {
        karr_next = S.k_out;
        for (int i = e; i < bounds[sgi + 2]; i++) karr_next = std::max(karr_next, sched[i]);
      }
      if (!S.last) {
        const size_t need = store_bytes(dp, S, n_in, S.k_out);
        if (need > p->seg_bytes[1 - cur]) {
          cudaFree(p->seg_pool[1 - cur]);
          p->seg_pool[1 - cur] = nullptr;
          p->seg_bytes[1 - cur] = 0;
          FS_CUDA_TRY(cudaMalloc(&p->seg_pool[1 - cur], need));
          p->seg_bytes[1 - cur] = need;
        }
        S.out = carve_store(p->seg_pool[1 - cur], S, n_in, S.k_out);
        S.out.shot_major = karr_next >= block_k ? 1 : 0;
        FS_CUDA_TRY(cudaMemsetAsync(d_nout, 0, 4, stream));
      }
      S.n_out = d_nout;
      int rc;
      if (karr >= block_k) rc = launch_block_kernel(p, a, S, karr, stream);
      else if (lseg_ready(p, a, S)) rc = launch_lane_segment(p, a, S, stream);
      else rc = launch_general_kernel(p, a, S, true, karr, (n_in + 31) / 32, stream);
      if (rc) return rc;
      if (S.last) break;
      uint32_t n_out = 0;
      FS_CUDA_TRY(cudaMemcpyAsync(&n_out, d_nout, 4, cudaMemcpyDeviceToHost, stream));
      FS_CUDA_TRY(cudaStreamSynchronize(stream));
      p->seg_counts.push_back(n_out);
      if (n_out == 0) break;
      S.in = S.out;
      cur = 1 - cur;
      n_in = n_out;
    }
  }
  return FS_OK;
}

// program-specialised general kernel (0 < k_max <= 7, no PostSelect / MeasActive / Retire)
bool gjit_supported(const fs_prog* p) {
  if (p->dp.k_max < 1 || p->dp.k_max > 7) return false;
  for (int i = 0; i < p->dp.num_instrs; i++) {
    const int op = FS_OPCODE(p->h_instrs[(size_t)i * FS_INS_WORDS]);
    if (op == FS_OP_POSTSELECT || op == FS_OP_MEAS_ACTIVE || op == FS_OP_RETIRE) return false;
  }
  return true;
}

int ensure_gjit(fs_prog* p) {
  if (p->jit_state == 1) return FS_OK;
  if (p->jit_state == -1) return set_error(FS_ERR_ARG, p->jit_error);
  p->jit_state = -1;
  fsjit::GeneralKernelSource K = fsjit::gen_general_kernel(p->desc, p->h_instrs, p->h_gates, p->h_paulis,
                                                           p->h_reclists, p->h_record_out, p->h_bit_slot,
                                                           p->h_case_pauli_off, p->h_site_case_off, p->h_fparams);
  const int nw = K.arr_regs ? 4 : 2;
  const size_t fs_words = (size_t)(2 * p->dp.n + 3) / 4 * 4;
  const size_t smem = nw * fs_words * 4 + (K.arr_regs ? 0 : (size_t)nw * 32 * 16 * (((size_t)1 << K.cap_log2) - K.nreg));
  if (smem > kSmemBudget) { p->jit_error = "program too large for the specialised general kernel"; return FS_ERR_ARG; }
  std::string err = fsjit::compile(K.src, fsjit::self_dir() + "/../csrc", p->jit, "fs_jit_general");
  if (!err.empty()) { p->jit_error = err; return set_error(FS_ERR_ARG, err); }
  fsjit::Api& J = fsjit::api();
  if (J.cuFuncSetAttribute(p->jit.fn, 8, (int)smem) != 0) { p->jit_error = "cuFuncSetAttribute failed"; return FS_ERR_ARG; }
  FS_CUDA_TRY(cudaMalloc(&p->d_pslot, sizeof(uint16_t) * K.pslot.size()));
  FS_CUDA_TRY(cudaMemcpy(p->d_pslot, K.pslot.data(), sizeof(uint16_t) * K.pslot.size(), cudaMemcpyHostToDevice));
  p->jit_nblocks = K.nblocks;
  FS_CUDA_TRY(cudaMalloc(&p->d_site_block, sizeof(int) * K.site_block.size()));
  FS_CUDA_TRY(cudaMemcpy(p->d_site_block, K.site_block.data(), sizeof(int) * K.site_block.size(), cudaMemcpyHostToDevice));
  p->gjit_threads = nw * 32;
  p->gjit_smem = smem;
  p->jit_state = 1;
  return FS_OK;
}

// per-word fault lists for the specialised kernels (fs_jit_kernels.cuh fault_list_kernel)
int alloc_fault_lists(fs_prog* p, size_t W, uint32_t** fent, uint32_t** bcount, uint32_t** ntot) {
  const int nb = std::max(1, p->jit_nblocks);
  const uint32_t cap = (uint32_t)p->jit_stage;
  const size_t need = align_up((size_t)cap * W * 4, 256) + align_up((size_t)nb * W * 4, 256) + W * 4 + 256;
  if (need > p->flist_bytes) {
    cudaFree(p->flist);
    p->flist = nullptr;
    p->flist_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->flist, need));
    p->flist_bytes = need;
  }
  unsigned char* fb8 = static_cast<unsigned char*>(p->flist);
  *fent = reinterpret_cast<uint32_t*>(fb8);
  *bcount = reinterpret_cast<uint32_t*>(fb8 + align_up((size_t)cap * W * 4, 256));
  *ntot = reinterpret_cast<uint32_t*>(fb8 + align_up((size_t)cap * W * 4, 256) + align_up((size_t)nb * W * 4, 256));
  return FS_OK;
}

// fault lists of words [w0, w0 + nw) of the call
int run_fault_lists(fs_prog* p, const fs::RunArgs& a, size_t w0, size_t nw, uint32_t* fent, uint32_t* bcount,
                    uint32_t* ntot, cudaStream_t stream) {
  fs::fault_list_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, stream>>>(
      p->dp, a.seed, (a.shot0 >> 5) + w0, (uint32_t)nw, a.ostride, p->d_site_block, p->jit_nblocks, fent + w0,
      bcount + w0, ntot + w0, (uint32_t)p->jit_stage);
  p->launches++;
  FS_CUDA_TRY(cudaGetLastError());
  return FS_OK;
}


// ------------------------------------------------------------------ large-k plan
// Microcode of one fused pass (format in fs_hbm_fused.cuh).  `T` = the pass's 12 tile axes in
// tile-bit order (bits 8..11 = register bits), `base` = the live axes outside the tile.  The
// layout is static over the pass (D.Tf == D.T); a mixing instruction on a thread bit exchanges
// the tile through shared memory.  (Moving axes into register bits with half-tile swaps and
// farthest-next-use eviction was measured: config 3 has almost no reuse of thread-bit axes, and
// the swaps' per-thread register selects cost more than the exchanges they replace.)
void compile_pass_code(std::vector<fs::TileOp>& pops, const std::vector<int>& T, const std::vector<int>& base,
                       const std::vector<int>& lowq, fs::PassDesc& D, HbmPlan& PL) {
  D.code_off = (int)PL.code.size();
  D.const_off = (int)PL.consts.size();
  std::vector<uint32_t>& C = PL.code;
  int at[fs::kTileBits];
  std::vector<int> pos(64, -1);
  for (int i = 0; i < fs::kTileBits; i++) { at[i] = T[i]; pos[T[i]] = i; }
  for (size_t i = 0; i < base.size(); i++) pos[base[i]] = fs::kTileBits + (int)i;
  auto isreg = [](int x) { return x >= 8 && x < 12; };
  auto rmask = [](int R) { return (uint32_t)((0xFF00F0F0CCCCAAAAull >> (16 * R)) & 0xFFFFu); };
  auto mix_axis = [](const fs::TileOp& o) {
    return o.kind == fs::TO_CX ? o.pb : (o.kind == fs::TO_H || o.kind == fs::TO_EXPAND) ? o.pa : -1;
  };
  auto add_const = [&](const fs::TileOp& o) {
    fs::PassConst k{};
    k.c0 = o.c0; k.c1 = o.c1; k.c2 = o.c2; k.c3 = o.c3;
    k.instr = o.instr;
    k.kind = o.kind;
    PL.consts.push_back(k);
    return (uint32_t)(PL.consts.size() - 1 - D.const_off);
  };
  for (size_t i = 0; i < pops.size();) {
    fs::TileOp& o = pops[i];
    if (o.diag_run > 0) {
      uint32_t sv[32] = {0}, N[32] = {0}, M[4] = {0}, QQ = 0;
      std::vector<uint32_t> rots;
      for (int r = 0; r < o.diag_run; r++) {
        fs::TileOp& d = pops[i + r];
        d.la = (int8_t)pos[d.pa];
        d.lb = d.pb >= 0 ? (int8_t)pos[d.pb] : (int8_t)-1;
        if (d.kind == fs::TO_S) sv[d.la] += 1;
        else if (d.kind == fs::TO_SDAG) sv[d.la] += 3;
        else if (d.kind == fs::TO_CZ) {
          const int a = d.la, b = d.lb;
          if (!isreg(a) && !isreg(b)) N[std::min(a, b)] ^= 1u << std::max(a, b);
          else if (isreg(a) && !isreg(b)) M[a - 8] ^= 1u << b;
          else if (!isreg(a) && isreg(b)) M[b - 8] ^= 1u << a;
          else QQ ^= rmask(a - 8) & rmask(b - 8);
        } else {  // ROT
          rots.push_back((uint32_t)d.la | add_const(d) << 8);
        }
      }
      uint32_t lin0 = 0, lin1 = 0, sr = 0;
      for (int x = 0; x < 32; x++) {
        if (isreg(x)) { sr |= (sv[x] & 3u) << (2 * (x - 8)); continue; }
        lin0 |= (sv[x] & 1u) << x;
        lin1 |= ((sv[x] >> 1) & 1u) << x;
      }
      std::vector<uint32_t> terms;
      for (int a2 = 0; a2 < 32; a2++)
        if (N[a2]) { terms.push_back((uint32_t)a2); terms.push_back(N[a2]); }
      const uint32_t nterm = (uint32_t)terms.size() / 2;
      C.push_back(fs::MC_DIAG | nterm << 4 | (uint32_t)rots.size() << 12);
      C.push_back(lin0);
      C.push_back(lin1);
      for (int R = 0; R < 4; R++) C.push_back(M[R]);
      C.push_back(sr | QQ << 16);
      C.insert(C.end(), terms.begin(), terms.end());
      C.insert(C.end(), rots.begin(), rots.end());
      i += o.diag_run;
      continue;
    }
    const int q = mix_axis(o);
    const uint32_t m = (uint32_t)pos[q];
    o.la = (int8_t)pos[o.pa];
    o.lb = o.pb >= 0 ? (int8_t)pos[o.pb] : (int8_t)-1;
    if (o.kind == fs::TO_H) C.push_back(fs::MC_H | m << 4);
    else if (o.kind == fs::TO_CX) C.push_back(fs::MC_CX | m << 4 | (uint32_t)pos[o.pa] << 9);
    else C.push_back(fs::MC_EXP | m << 4 | add_const(o) << 16);  // EXPAND
    i++;
  }
  for (int i = 0; i < fs::kTileBits; i++) D.Tf[i] = (int8_t)at[i];
  for (int j = 0; j < fs::kTileElems; j++) {
    uint32_t g = 0;
    for (int b = 0; b < fs::kTileBits - 8; b++) g |= (uint32_t)((j >> b) & 1) << at[8 + b];
    D.dep_hi_f[j] = g;
  }
  D.ncode = (int)PL.code.size() - D.code_off;
  D.nconst = (int)PL.consts.size() - D.const_off;
}

// Host walk of the program (shot-independent): logical->physical axis map, the scalar
// segments, per-instruction array kernels, measurements, and -- when the live dimension is at
// least fs::kTileBits -- fused tile passes (fs_hbm_fused.cuh).
int plan_hbm(fs_prog* p, int stop, bool fused, const std::vector<int>& cuts) {
  HbmPlan& PL = p->hplan;
  if (PL.built && PL.stop == stop && PL.fused == fused && PL.cuts == cuts) return FS_OK;
  PL = HbmPlan{};
  PL.stop = stop;
  PL.fused = fused;
  PL.cuts = cuts;
  p->pass_jit = 0;
  p->pass_fn.clear();
  const fs::DevProg& dp = p->dp;
  const int* ins_all = p->h_instrs.data();
  const double* fpar = p->h_fparams.data();
  std::vector<int> live;
  auto is_live = [&](int q) { return std::find(live.begin(), live.end(), q) != live.end(); };
  auto dead_list = [&](std::initializer_list<int> extra) {
    fs::DeadBits d{};
    int top = -1;
    for (int x : live) top = std::max(top, x);
    for (int x : extra) top = std::max(top, x);
    std::vector<int> pos;
    for (int q = 0; q <= top; q++) {
      const bool ise = std::find(extra.begin(), extra.end(), q) != extra.end();
      if (!is_live(q) || ise) pos.push_back(q);
    }
    std::sort(pos.begin(), pos.end());
    pos.erase(std::unique(pos.begin(), pos.end()), pos.end());
    d.n = (int)pos.size();
    for (int t = 0; t < d.n; t++) d.pos[t] = (int8_t)pos[t];
    return d;
  };
  auto lowest_dead = [&]() {
    for (int q = 0; q < dp.k_max; q++)
      if (!is_live(q)) return q;
    return -1;
  };
  auto cpx = [&](int off) { return make_double2(fpar[off], fpar[off + 1]); };
  // pending fused pass
  std::vector<fs::TileOp> pops;
  std::vector<int> need;
  bool code_overflow = false;
  auto flush = [&]() {
    if (pops.empty()) return;
    fs::PassDesc D{};
    std::vector<int> T = need;
    for (int q = 0; q < 3; q++)
      if (is_live(q) && std::find(T.begin(), T.end(), q) == T.end()) T.push_back(q);
    for (int q = 0; (int)T.size() < fs::kTileBits && q < 64; q++)
      if (is_live(q) && std::find(T.begin(), T.end(), q) == T.end()) T.push_back(q);
    // layout: live low physical axes 0..2 on thread bits 0..2 (128-byte coalesced accesses),
    // the four most-mixed other axes on the register bits 8..11, the rest on thread bits
    std::vector<int> lowq;
    for (int q : T)
      if (q < 3 && is_live(q)) lowq.push_back(q);
    std::sort(lowq.begin(), lowq.end());
    std::vector<std::pair<int, int>> use;  // (-mixing uses, axis)
    for (int q : T) {
      if (std::find(lowq.begin(), lowq.end(), q) != lowq.end()) continue;
      int cnt = 0;
      for (auto& o : pops) {
        const int mix = o.kind == fs::TO_CX ? o.pb : (o.kind == fs::TO_H || o.kind == fs::TO_EXPAND) ? o.pa : -1;
        cnt += mix == q;
      }
      use.push_back({-cnt, q});
    }
    std::sort(use.begin(), use.end());
    std::vector<int> regs, thr;
    for (auto& u : use) (regs.size() < 4 ? regs : thr).push_back(u.second);
    std::sort(thr.begin(), thr.end());
    T.clear();
    T.insert(T.end(), lowq.begin(), lowq.end());
    T.insert(T.end(), thr.begin(), thr.end());
    T.insert(T.end(), regs.begin(), regs.end());
    if ((int)T.size() != fs::kTileBits) { pops.clear(); need.clear(); return; }  // cannot happen (k >= kTileBits)
    for (int i = 0; i < fs::kTileBits; i++) D.T[i] = (int8_t)T[i];
    std::vector<int> base;
    for (int q : live)
      if (std::find(T.begin(), T.end(), q) == T.end()) base.push_back(q);
    std::sort(base.begin(), base.end());
    D.nbase = (int)base.size();
    for (int i = 0; i < D.nbase; i++) D.base[i] = (int8_t)base[i];
    for (int j = 0; j < fs::kTileElems; j++) {
      uint32_t g = 0;
      for (int b = 0; b < fs::kTileBits - 8; b++) g |= (uint32_t)((j >> b) & 1) << T[8 + b];
      D.dep_hi[j] = g;
    }
    auto diag = [](int k) { return k == fs::TO_S || k == fs::TO_SDAG || k == fs::TO_CZ || k == fs::TO_ROT; };
    for (size_t i = 0; i < pops.size();) {
      if (!diag(pops[i].kind)) { pops[i].diag_run = 0; i++; continue; }
      size_t e = i;
      while (e < pops.size() && diag(pops[e].kind)) e++;
      for (size_t r = i; r < e; r++) pops[r].diag_run = 0;
      pops[i].diag_run = (int8_t)std::min<size_t>(e - i, 127);
      i = i + std::min<size_t>(e - i, 127);
    }
    compile_pass_code(pops, T, base, lowq, D, PL);
    if (D.ncode > fs::kPassMaxCode || D.nconst > fs::kPassMaxOps) code_overflow = true;
    D.nops = (int)pops.size();
    D.op_off = (int)PL.tileops.size();
    PL.tileops.insert(PL.tileops.end(), pops.begin(), pops.end());
    HbmStep st{};
    st.kind = HbmStep::PASS;
    st.pass = (int)PL.passes.size();
    PL.passes.push_back(D);
    PL.steps.push_back(st);
    pops.clear();
    need.clear();
  };
  auto arr = [&](const fs::ArrOp& o, uint64_t count) {
    HbmStep st{};
    st.kind = HbmStep::ARR;
    st.op = o;
    st.count = count;
    PL.steps.push_back(st);
  };
  // checkpoint c (state after instructions [0, c)): every step before it is complete, then a
  // DUMP step records the frames / gamma / active array with the axis map of that point
  size_t next_cut = 0;
  auto dump_at = [&](int pos) {
    while (next_cut < cuts.size() && cuts[next_cut] == pos) {
      flush();
      HbmStep st{};
      st.kind = HbmStep::DUMP;
      st.i0 = pos;
      st.cp = (int)next_cut;
      st.i1 = (int)live.size();
      for (int b = 0; b < (int)live.size(); b++) st.map.phys[b] = (int8_t)live[b];
      PL.steps.push_back(st);
      next_cut++;
    }
  };
  auto next_cut_after = [&](int pos) {
    for (size_t c = next_cut; c < cuts.size(); c++)
      if (cuts[c] > pos) return cuts[c];
    return INT_MAX;
  };
  int i = 0;
  dump_at(0);
  while (i < stop) {
    int j = i;
    while (j < stop) {
      const int op = FS_OPCODE(ins_all[(size_t)j * FS_INS_WORDS]);
      if (op == FS_OP_MEAS_ACTIVE || op == FS_OP_MEAS_COLLAPSE) break;
      j++;
    }
    // a checkpoint inside [i, j) ends this range there (the rest is the next iteration's)
    const int jc = std::min(j, next_cut_after(i));
    const bool cut_here = jc < j;
    j = jc;
    if (j > i) {
      HbmStep st{};
      st.kind = HbmStep::SCALAR;
      st.i0 = i;
      st.i1 = j;
      PL.steps.push_back(st);
    }
    for (int t = i; t < j; t++) {
      const int* I = ins_all + (size_t)t * FS_INS_WORDS;
      const int op = FS_OPCODE(I[0]);
      if (op != FS_OP_ARRAY_GATE && op != FS_OP_EXPAND && op != FS_OP_ARRAY_ROT && op != FS_OP_RETIRE) continue;
      const int k_after = p->h_sched[t];
      // candidate for a fused pass?
      if (fused && op != FS_OP_RETIRE && k_after >= fs::kTileBits && k_after <= 31 &&
          (int)live.size() + (op == FS_OP_EXPAND) >= fs::kTileBits) {
        fs::TileOp to{};
        to.instr = t;
        to.pa = to.pb = -1;
        int mix = -1;
        if (op == FS_OP_ARRAY_GATE) {
          const int g = I[1];
          to.pa = (int8_t)live[I[4]];
          if (g == FS_G_CX || g == FS_G_CZ) to.pb = (int8_t)live[I[5]];
          to.kind = g == FS_G_H ? fs::TO_H : g == FS_G_S ? fs::TO_S : g == FS_G_SDAG ? fs::TO_SDAG
                  : g == FS_G_CX ? fs::TO_CX : fs::TO_CZ;
          if (g == FS_G_H) mix = to.pa;
          if (g == FS_G_CX) mix = to.pb;
        } else if (op == FS_OP_ARRAY_ROT) {
          to.kind = fs::TO_ROT;
          to.pa = (int8_t)live[I[2]];
          to.c0 = cpx(I[5]);
          to.c1 = cpx(I[5] + 2);
        } else {  // EXPAND onto the lowest dead physical axis
          to.kind = fs::TO_EXPAND;
          to.pa = (int8_t)lowest_dead();
          mix = to.pa;
          to.c0 = cpx(I[5]); to.c1 = cpx(I[5] + 2); to.c2 = cpx(I[5] + 4); to.c3 = cpx(I[5] + 6);
        }
        if ((int)pops.size() >= fs::kPassMaxOps) flush();
        if (mix >= 0 && std::find(need.begin(), need.end(), mix) == need.end()) {
          int low = 0;
          for (int q = 0; q < 3; q++)
            if ((is_live(q) || q == mix) && std::find(need.begin(), need.end(), q) == need.end() && q != mix) low++;
          if ((int)need.size() + 1 + low > fs::kTileBits) flush();
          need.push_back(mix);
        }
        pops.push_back(to);
        if (op == FS_OP_EXPAND) live.push_back(to.pa);
        continue;
      }
      flush();
      fs::ArrOp o{};
      o.instr = t;
      if (op == FS_OP_ARRAY_GATE) {
        const int g = I[1], k = I[6];
        o.pa = live[I[4]];
        if (g == FS_G_CX || g == FS_G_CZ) {
          o.pb = live[I[5]];
          o.kind = g == FS_G_CX ? fs::HA_CX : fs::HA_CZ;
          o.dead = dead_list({o.pa, o.pb});
          arr(o, 1ull << (k - 2));
        } else {
          o.kind = g == FS_G_H ? fs::HA_H : (g == FS_G_S ? fs::HA_S : fs::HA_SDAG);
          o.dead = dead_list({o.pa});
          arr(o, 1ull << (k - 1));
        }
      } else if (op == FS_OP_EXPAND) {
        const int kb = I[6];
        o.kind = fs::HA_EXPAND;
        o.pa = lowest_dead();
        o.dead = dead_list({o.pa});
        o.c0 = cpx(I[5]); o.c1 = cpx(I[5] + 2); o.c2 = cpx(I[5] + 4); o.c3 = cpx(I[5] + 6);
        arr(o, 1ull << kb);
        live.push_back(o.pa);
      } else if (op == FS_OP_ARRAY_ROT) {
        const int k = I[6];
        o.kind = fs::HA_ROT;
        o.pa = live[I[2]];
        o.dead = dead_list({o.pa});
        o.c0 = cpx(I[5]); o.c1 = cpx(I[5] + 2);
        arr(o, 1ull << (k - 1));
      } else {  // RETIRE
        const int k = I[6];
        o.kind = fs::HA_RETIRE;
        o.pa = live[I[2]];
        o.dead = dead_list({o.pa});
        arr(o, 1ull << (k - 1));
        live.erase(live.begin() + I[2]);
      }
    }
    flush();
    if (cut_here) {
      dump_at(j);
      i = j;
      continue;
    }
    dump_at(j);
    if (j >= stop) { i = j; break; }
    const int* I = ins_all + (size_t)j * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]);
    const int k = I[6];
    HbmStep st{};
    st.kind = HbmStep::MEAS;
    st.i0 = j;
    st.op.instr = j;
    st.op.pa = live[I[2]];
    st.op.dead = dead_list({st.op.pa});
    st.count = 1ull << (k - 1);
    st.collapse = op == FS_OP_MEAS_COLLAPSE ? 1 : 0;
    st.u10 = make_double2(0, 0);
    st.u11 = make_double2(1, 0);
    if (st.collapse) { st.u10 = cpx(I[5] + 4); st.u11 = cpx(I[5] + 6); }
    PL.steps.push_back(st);
    if (st.collapse) live.erase(live.begin() + I[2]);
    i = j + 1;
    dump_at(i);
  }
  const int kst = stop > 0 ? p->h_sched[stop - 1] : 0;
  if ((int)live.size() != kst) return set_error(FS_ERR_ARG, "internal: axis map out of sync with schedule");
  PL.final_live = live;
  if (code_overflow) return set_error(FS_ERR_ARG, "internal: fused pass microcode exceeds its shared-memory area");
  cudaFree(p->d_passes);
  cudaFree(p->d_tileops);
  cudaFree(p->d_code);
  cudaFree(p->d_consts);
  p->d_passes = nullptr;
  p->d_tileops = nullptr;
  p->d_code = nullptr;
  p->d_consts = nullptr;
  if (!PL.code.empty()) {
    FS_CUDA_TRY(cudaMalloc(&p->d_code, sizeof(uint32_t) * PL.code.size()));
    FS_CUDA_TRY(cudaMemcpy(p->d_code, PL.code.data(), sizeof(uint32_t) * PL.code.size(), cudaMemcpyHostToDevice));
  }
  if (!PL.consts.empty()) {
    FS_CUDA_TRY(cudaMalloc(&p->d_consts, sizeof(fs::PassConst) * PL.consts.size()));
    FS_CUDA_TRY(cudaMemcpy(p->d_consts, PL.consts.data(), sizeof(fs::PassConst) * PL.consts.size(), cudaMemcpyHostToDevice));
  }
  if (!PL.passes.empty()) {
    FS_CUDA_TRY(cudaMalloc(&p->d_passes, sizeof(fs::PassDesc) * PL.passes.size()));
    FS_CUDA_TRY(cudaMemcpy(p->d_passes, PL.passes.data(), sizeof(fs::PassDesc) * PL.passes.size(), cudaMemcpyHostToDevice));
    FS_CUDA_TRY(cudaMalloc(&p->d_tileops, sizeof(fs::TileOp) * PL.tileops.size()));
    FS_CUDA_TRY(cudaMemcpy(p->d_tileops, PL.tileops.data(), sizeof(fs::TileOp) * PL.tileops.size(), cudaMemcpyHostToDevice));
  }
  PL.built = true;
  return FS_OK;
}

// ------------------------------------------------------------------ specialised pass kernels
// Each fused pass's microcode compiled to straight-line code (NVRTC): masks, register bits,
// exchange partners and address deposits become constants; the interpreter
// (fs_hbm_fused.cuh hbm_fused_pass_kernel) remains the fallback (FS_HBM_NO_JIT).
std::string gen_pass_source(const HbmPlan& PL, bool tma_ok) {
  std::ostringstream o;
  o << "#include \"fs_hbm_fused.cuh\"\nusing namespace fs;\n";
  auto hexu = [](uint32_t x) {
    std::ostringstream t;
    t << "0x" << std::hex << x << "u";
    return t.str();
  };
  for (size_t pi = 0; pi < PL.passes.size(); pi++) {
    const fs::PassDesc& D = PL.passes[pi];
    // TMA staging when the tile's lowest L >= 3 bits are physical axes 0..L-1: the tile is
    // 2^(12-L) contiguous runs of 2^L amplitudes (16 << L bytes), one bulk copy each
    int L = 0;
    while (L < 8 && D.T[L] == L) L++;
    const bool tma = tma_ok && L >= 3;
    const int nseg = 1 << (fs::kTileBits - L), segb = 16 << L;
    // smem: exchange half-buffer (32 KiB) | next-tile staging (64 KiB) | resolved constants
    o << "extern \"C\" __global__ void __launch_bounds__(256, 2) fs_pass_" << pi
      << "(HbmState H, const PassConst* __restrict__ consts, uint32_t W) {\n"
      << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
      << "  double2* T = reinterpret_cast<double2*>(smem_raw);\n"
      << "  double2* Sg = reinterpret_cast<double2*>(smem_raw + " << (8 << fs::kTileBits) << ");\n"
      << "  double2* cs = reinterpret_cast<double2*>(smem_raw + " << (24 << fs::kTileBits) << ");\n"
      << "  const uint32_t shot = blockIdx.y, w = shot >> 5, bit = 1u << (shot & 31);\n"
      << "  if (!(H.alive[w] & bit)) return;\n"
      << "  const uint32_t tid = threadIdx.x;\n";
    if (D.nconst)
      o << "  for (int i = tid; i < " << D.nconst << "; i += 256) {\n"
        << "    const PassConst& k = consts[" << D.const_off << " + i];\n"
        << "    const bool par = (H.par[(size_t)k.instr * W + w] & bit) != 0;\n"
        << "    double2 a = k.c0, b = k.c1;\n"
        << "    if (par) { if (k.kind == TO_ROT) { a = k.c1; b = k.c0; } else { a = k.c2; b = k.c3; } }\n"
        << "    cs[2 * i] = a;\n    cs[2 * i + 1] = b;\n  }\n";
    o << "  const uint32_t dep_lo = 0u";
    for (int i = 0; i < 8; i++) o << " | (((tid >> " << i << ") & 1u) << " << (int)D.T[i] << ")";
    o << ";\n  const uint32_t dep_lo_f = 0u";
    for (int i = 0; i < 8; i++) o << " | (((tid >> " << i << ") & 1u) << " << (int)D.Tf[i] << ")";
    auto deposit = [&](const char* t) {
      std::ostringstream d;
      d << "0ull";
      for (int i = 0; i < D.nbase; i++) d << " | ((uint64_t)((" << t << " >> " << i << ") & 1u) << " << (int)D.base[i] << ")";
      return d.str();
    };
    auto prefetch = [&](const char* basevar) {  // this thread's 16 elements of a tile -> its Sg slots
      if (tma) {  // segment s (local index s << L + [0, 2^L)): threads tid < nseg, s = tid + 256 r
        o << "      if (tid == 0) mbar_expect_tx(&bar, " << (16u << fs::kTileBits) << "u);\n"
          << "      fence_proxy_async_smem();\n";
        if (nseg < 256) o << "      if (tid < " << nseg << "u) ";
        else o << "      ";
        o << "bulk_g2s(Sg + (tid << " << L << "), A + (" << basevar << " | seg_lo), " << segb << "u, &bar);\n";
        for (int r = 1; r < nseg / 256; r++) {  // segments tid + 256 r: local bits L + 8.. from r
          uint32_t hi = 0;
          for (int b = 0; L + 8 + b < fs::kTileBits; b++)
            if ((r >> b) & 1) hi |= 1u << D.T[L + 8 + b];
          o << "      bulk_g2s(Sg + ((tid + " << 256 * r << "u) << " << L << "), A + (" << basevar << " | seg_lo | " << hexu(hi)
            << "), " << segb << "u, &bar);\n";
        }
        return;
      }
      for (int j = 0; j < fs::kTileElems; j++)
        o << "      cp_async16(Sg + tid + " << 256 * j << ", A + (" << basevar << " | dep_lo | " << hexu(D.dep_hi[j]) << "));\n";
      o << "      cp_async_commit();\n";
    };
    if (tma) {  // segment s: local bits L.. = s bits on axes T[L..]; tid supplies s bits 0..7
      o << ";\n  const uint32_t seg_lo = 0u";
      for (int i = 0; i < 8 && L + i < fs::kTileBits; i++) o << " | (((tid >> " << i << ") & 1u) << " << (int)D.T[L + i] << ")";
      o << ";\n  __shared__ uint64_t bar;\n  uint32_t phase = 0u;\n"
        << "  if (tid == 0) { mbar_init(&bar, 1u); asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\"); }\n";
    }
    o << ";\n  __syncthreads();\n"
      << "  double2* __restrict__ A = H.amps + (size_t)shot * H.cap;\n"
      << "  double2 v[16];\n"
      << "  const uint32_t NT = " << (1u << D.nbase) << "u;\n"
      << "  if (blockIdx.x < NT) {\n    const uint64_t b0 = " << deposit("blockIdx.x") << ";\n";
    prefetch("b0");
    o << "  }\n"
      << "  for (uint32_t ti = blockIdx.x; ti < NT; ti += gridDim.x) {\n"
      << "    const uint64_t base = " << deposit("ti") << ";\n"
      << "    const uint32_t X0 = tid | (ti << " << fs::kTileBits << ");\n";
    if (tma) o << "    mbar_wait(&bar, phase);\n    phase ^= 1u;\n";
    else o << "    cp_async_wait_all();\n";
    for (int j = 0; j < fs::kTileElems; j++) o << "    v[" << j << "] = Sg[tid + " << 256 * j << "];\n";
    if (tma) o << "    __syncthreads();  // every read of Sg before the next tile's bulk copies overwrite it\n";
    o << "    if (ti + gridDim.x < NT) {\n      const uint32_t tn = ti + gridDim.x;\n      const uint64_t bn = " << deposit("tn") << ";\n";
    prefetch("bn");
    o << "    }\n";
    const uint32_t* C = PL.code.data() + D.code_off;
    for (int pc = 0; pc < D.ncode;) {
      const uint32_t ow = C[pc];
      const uint32_t kind = ow & 15u;
      if (kind == fs::MC_DIAG) {
        const int nterm = (ow >> 4) & 0xFF, nrot = (ow >> 12) & 0xFF;
        const uint32_t lin0 = C[pc + 1], lin1 = C[pc + 2], sr = C[pc + 7];
        o << "    {\n      uint32_t e0 = 0u";
        if (lin0) o << " + __popc(X0 & " << hexu(lin0) << ")";
        if (lin1) o << " + 2u * __popc(X0 & " << hexu(lin1) << ")";
        o << ";\n";
        if (nterm) {
          o << "      uint32_t q = 0u";
          for (int t = 0; t < nterm; t++)
            o << " + ((X0 >> " << C[pc + 8 + 2 * t] << ") & 1u) * __popc(X0 & " << hexu(C[pc + 9 + 2 * t]) << ")";
          o << ";\n      e0 += 2u * q;\n";
        }
        o << "      const uint32_t eR[4] = {";
        for (int R = 0; R < 4; R++) {
          o << ((sr >> (2 * R)) & 3u) << "u";
          if (C[pc + 3 + R]) o << " + 2u * __popc(X0 & " << hexu(C[pc + 3 + R]) << ")";
          o << (R < 3 ? ", " : "};\n");
        }
        o << "      uint32_t Lm, Hm;\n      ipow_planes(e0, eR, " << hexu(sr >> 16) << ", Lm, Hm);\n"
          << "      apply_ipow(v, Lm, Hm);\n";
        if (nrot) {
          uint32_t rreg = 0;
          o << "      double2 g = make_double2(1, 0);\n"
            << "      double2 d[4] = {make_double2(1, 0), make_double2(1, 0), make_double2(1, 0), make_double2(1, 0)};\n";
          for (int r = 0; r < nrot; r++) {
            const uint32_t rw = C[pc + 8 + 2 * nterm + r];
            const int xa = rw & 31, k = rw >> 8;
            if (xa >= 8 && xa < 12) {
              o << "      g = cmul(g, cs[" << 2 * k << "]);\n      d[" << xa - 8 << "] = cmul(d[" << xa - 8
                << "], cdiv(cs[" << 2 * k + 1 << "], cs[" << 2 * k << "]));\n";
              rreg |= 1u << (xa - 8);
            } else {
              o << "      g = cmul(g, ((X0 >> " << xa << ") & 1u) ? cs[" << 2 * k + 1 << "] : cs[" << 2 * k << "]);\n";
            }
          }
          o << "      apply_rot(v, g, d, " << rreg << "u);\n";
        }
        o << "    }\n";
        pc += 8 + 2 * nterm + nrot;
        continue;
      }
      pc++;
      const int m = (ow >> 4) & 15;
      const int xa = (ow >> 9) & 31, k = (int)(ow >> 16);
      if (m >= 8) {
        const int R = m - 8;
        if (kind == fs::MC_H) {
          o << "    reg_h<" << R << ">(v);\n";
        } else if (kind == fs::MC_CX) {
          if (xa >= 8 && xa < 12) o << "    reg_cx<" << R << ">(v, 0, " << xa - 8 << ", tid, 0);\n";
          else o << "    if ((X0 >> " << xa << ") & 1u) reg_cx<" << R << ">(v, 3, 1, tid, 0);\n";
        } else {
          o << "    reg_expand<" << R << ">(v, cs[" << 2 * k << "], cs[" << 2 * k + 1 << "]);\n";
        }
        continue;
      }
      if (m < 5) {
        if (kind == fs::MC_H) o << "    xlane_h(v, tid, " << m << ");\n";
        else if (kind == fs::MC_CX) o << "    xlane_cx(v, " << m << ", cx_ctl_mask(" << xa << ", X0));\n";
        else o << "    xlane_exp(v, tid, " << m << ", cs[" << 2 * k << "], cs[" << 2 * k + 1 << "]);\n";
      } else {
        if (kind == fs::MC_H) o << "    xsmem_half<0>(v, T, tid, " << m << ", 0u, make_double2(1, 0), make_double2(1, 0));\n";
        else if (kind == fs::MC_CX) o << "    xsmem_half<1>(v, T, tid, " << m << ", cx_ctl_mask(" << xa << ", X0), make_double2(1, 0), make_double2(1, 0));\n";
        else o << "    xsmem_half<2>(v, T, tid, " << m << ", 0u, cs[" << 2 * k << "], cs[" << 2 * k + 1 << "]);\n";
      }
    }
    for (int j = 0; j < fs::kTileElems; j++) o << "    A[base | dep_lo_f | " << hexu(D.dep_hi_f[j]) << "] = v[" << j << "];\n";
    o << "  }\n}\n";
  }
  return o.str();
}

int ensure_pass_jit(fs_prog* p) {
  if (p->pass_jit == 1) return FS_OK;
  if (p->pass_jit == -1) return FS_ERR_ARG;
  p->pass_jit = -1;
  const HbmPlan& PL = p->hplan;
  const std::string src = gen_pass_source(PL, p->env.pass_tma);
  // one module per distinct source per process (tests and benches create many programs)
  // (modules belong to a context: the key is (current context, source))
  static std::mutex mu;
  static std::map<std::pair<fsjit::CUcontext, std::string>, fsjit::CUmodule> cache;
  std::lock_guard<std::mutex> g(mu);
  fsjit::Api& J = fsjit::api();
  if (!J.ok) { p->pass_jit_err = J.why; return FS_ERR_ARG; }
  fsjit::CUcontext ctx = nullptr;
  J.cuCtxGetCurrent(&ctx);
  const auto key = std::make_pair(ctx, src);
  fsjit::CUmodule mod = nullptr;
  auto it = cache.find(key);
  if (it != cache.end()) {
    mod = it->second;
  } else {
    fsjit::Compiled c;
    std::string err = fsjit::compile(src, fsjit::self_dir() + "/../csrc", c, "fs_pass_0");
    if (!err.empty()) { p->pass_jit_err = err; return FS_ERR_ARG; }
    mod = c.mod;
    cache[key] = mod;
  }
  p->pass_fn.assign(PL.passes.size(), nullptr);
  for (size_t i = 0; i < PL.passes.size(); i++) {
    const std::string name = "fs_pass_" + std::to_string(i);
    if (J.cuModuleGetFunction(&p->pass_fn[i], mod, name.c_str()) != 0) { p->pass_jit_err = "missing " + name; return FS_ERR_ARG; }
    const int smem = (24 << fs::kTileBits) + 32 * std::max(PL.passes[i].nconst, 1);
    if (J.cuFuncSetAttribute(p->pass_fn[i], 8, smem) != 0) { p->pass_jit_err = "cuFuncSetAttribute"; return FS_ERR_ARG; }
  }
  p->pass_jit = 1;
  return FS_OK;
}

// ------------------------------------------------------------------ large-k engine driver
int launch_hbm(fs_prog* p, fs::RunArgs& a, cudaStream_t stream) {
  const fs::DevProg& dp = p->dp;
  const uint64_t cap = 1ull << dp.k_max;
  const size_t per_shot = cap * sizeof(double2);
  const int n = dp.n, S = dp.num_slots, O = dp.O, N = dp.num_instrs;
  const int nblk = 64;
  size_t free_b = 0, total_b = 0;
  FS_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  auto state_bytes = [&](uint64_t B) {
    const uint64_t Wm = (B + 31) / 32;
    size_t b = 0;
    b += align_up(B * per_shot, 256);
    b += align_up(4 * Wm * (2 * (size_t)n + S + O + 5 + (size_t)N), 256);
    b += align_up(B * (16 + 4 + 2 * nblk * 8 + 16 + 32), 256);
    return b + 4096;
  };
  uint64_t want = (a.nshots + 31) / 32 * 32;
  const size_t budget = std::min<size_t>((size_t)((double)(free_b + p->hbm_bytes) * 0.80), (size_t)140 << 30);
  uint64_t B = want;
  while (B > 32 && state_bytes(B) > budget) B = std::max<uint64_t>(32, (B / 2) / 32 * 32);
  if (state_bytes(B) > budget) {
    if (a.nshots <= 1 && state_bytes(1) <= budget) B = 1;
    else return set_error(FS_ERR_ARG, "active array too large for device memory");
  }
  if (state_bytes(B) > p->hbm_bytes) {
    cudaFree(p->hbm);
    p->hbm = nullptr;
    p->hbm_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->hbm, state_bytes(B)));
    p->hbm_bytes = state_bytes(B);
  }
  const uint64_t Wm = (B + 31) / 32;
  fs::HbmState H{};
  {
    Stage st;
    st.base = static_cast<unsigned char*>(p->hbm);
    H.amps = st.take<double2>(B * cap);
    H.fx = st.take<uint32_t>(Wm * n + 1);
    H.fz = st.take<uint32_t>(Wm * n + 1);
    H.slots = st.take<uint32_t>(Wm * S + 1);
    H.obs = st.take<uint32_t>(Wm * O + 1);
    H.alive = st.take<uint32_t>(Wm);
    H.err = st.take<uint32_t>(Wm);
    H.brw = st.take<uint32_t>(Wm);
    H.frozen = st.take<uint32_t>(Wm);
    H.par = st.take<uint32_t>(Wm * N + 1);
    H.gamma = st.take<double2>(B);
    H.smcount = st.take<uint32_t>(B);
    H.red = st.take<double>(B * 2 * nblk);
    H.p1 = st.take<double>(B);
    H.pall = st.take<double>(B);
    H.kco = st.take<double2>(2 * B);
    H.cap = cap;
    H.nblk = nblk;
  }
  // all output words are written by the scalar kernel unless a batch halts early
  if (dp.U) FS_CUDA_TRY(cudaMemsetAsync(a.meas, 0, sizeof(uint32_t) * dp.U * (size_t)a.W, stream));
  if (dp.D) FS_CUDA_TRY(cudaMemsetAsync(a.det, 0, sizeof(uint32_t) * dp.D * (size_t)a.W, stream));
  const bool splitmix = a.flags & FS_RNG_SPLITMIX;
  auto scalar = [&](int i0, int i1, int init, uint64_t batch0, uint32_t W) -> int {
    dim3 g((W + 127) / 128);
    if (splitmix) fs::hbm_scalar_kernel<true><<<g, 128, 0, stream>>>(dp, a, H, i0, i1, init, batch0, W);
    else fs::hbm_scalar_kernel<false><<<g, 128, 0, stream>>>(dp, a, H, i0, i1, init, batch0, W);
    p->launches++;
    FS_CUDA_TRY(cudaGetLastError());
    return FS_OK;
  };
  const bool fused = !(a.flags & FS_FORCE_HBM) || p->env.hbm_fused;
  static const std::vector<int> no_cuts;
  int rc0 = plan_hbm(p, a.stop, fused && !p->env.hbm_unfused, a.ncp ? p->cp_list : no_cuts);
  if (rc0) return rc0;
  const HbmPlan& PL = p->hplan;
  const size_t pass_smem = fs::kPassSmem;
  const bool use_pass_jit = !PL.passes.empty() && !p->env.hbm_no_jit && ensure_pass_jit(p) == FS_OK;
  if (!PL.passes.empty())
    FS_CUDA_TRY(cudaFuncSetAttribute(fs::hbm_fused_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem));
  for (uint64_t batch0 = 0; batch0 < a.nshots; batch0 += B) {
    const uint64_t nb = std::min<uint64_t>(B, a.nshots - batch0);
    const uint32_t W = (uint32_t)((nb + 31) / 32);
    int rc = scalar(0, 0, 1, batch0, W);
    if (rc) return rc;
    fs::hbm_init_amps_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, stream>>>(H, (uint32_t)nb);
    p->launches++;
    auto run_op = [&](const fs::ArrOp& o, uint64_t count) -> int {
      if (count == 0) return FS_OK;
      const uint64_t want_x = (count + 255) / 256;
      const uint64_t gx = std::max<uint64_t>(1, std::min<uint64_t>(want_x, std::max<uint64_t>(1, 16384 / nb)));
      fs::hbm_array_kernel<<<dim3((unsigned)gx, (unsigned)nb), 256, 0, stream>>>(o, H, count, W);
      p->launches++;
      FS_CUDA_TRY(cudaGetLastError());
      return FS_OK;
    };
    for (const HbmStep& st : PL.steps) {
      switch (st.kind) {
        case HbmStep::SCALAR:
          if ((rc = scalar(st.i0, st.i1, 0, batch0, W))) return rc;
          break;
        case HbmStep::ARR:
          if ((rc = run_op(st.op, st.count))) return rc;
          break;
        case HbmStep::PASS: {
          const uint64_t ntiles = 1ull << PL.passes[st.pass].nbase;
          const uint64_t gx = std::max<uint64_t>(1, std::min<uint64_t>(ntiles, std::max<uint64_t>(1, 4096 / nb)));
          kt_begin(p, stream);
          if (use_pass_jit) {
            const fs::PassConst* cp = p->d_consts;
            uint32_t Wv = W;
            void* args[] = {&H, &cp, &Wv};
            const int smem = (24 << fs::kTileBits) + 32 * std::max(PL.passes[st.pass].nconst, 1);
            if (fsjit::api().cuLaunchKernel(p->pass_fn[st.pass], (unsigned)gx, (unsigned)nb, 1, fs::kTileThreads, 1, 1,
                                            (unsigned)smem, stream, args, nullptr) != 0)
              return set_error(FS_ERR_CUDA, "cuLaunchKernel(fs_pass) failed");
          } else {
            fs::hbm_fused_pass_kernel<<<dim3((unsigned)gx, (unsigned)nb), fs::kTileThreads, pass_smem, stream>>>(
                H, PL.passes[st.pass], p->d_code, p->d_consts, W);
          }
          kt_end(p, stream);
          p->launches++;
          FS_CUDA_TRY(cudaGetLastError());
          break;
        }
        case HbmStep::DUMP: {
          fs::hbm_cp_kernel<<<(W + 127) / 128, 128, 0, stream>>>(dp, a, H, batch0, W, st.cp);
          const uint64_t sz = 1ull << st.i1;
          const uint64_t gx = std::max<uint64_t>(1, std::min<uint64_t>((sz + 255) / 256, 1024));
          fs::hbm_gather_kernel<<<dim3((unsigned)gx, (unsigned)nb), 256, 0, stream>>>(
              dp, a, H, batch0, (uint32_t)nb, st.i1, st.map, a.cp_amps + 2 * p->cp_offs[st.cp]);
          p->launches += 2;
          FS_CUDA_TRY(cudaGetLastError());
          break;
        }
        case HbmStep::MEAS: {
          const int nbu = (int)std::max<uint64_t>(1, std::min<uint64_t>(nblk, (st.count + 2047) / 2048));
          fs::hbm_reduce_kernel<<<dim3(nbu, (unsigned)nb), 256, 0, stream>>>(st.op, H, st.count, st.collapse, st.u10, st.u11);
          fs::hbm_reduce_final_kernel<<<(unsigned)((nb + 127) / 128), 128, 0, stream>>>(H, (uint32_t)nb, nbu);
          p->launches += 2;
          FS_CUDA_TRY(cudaGetLastError());
          if ((rc = scalar(st.i0, st.i0 + 1, 0, batch0, W))) return rc;
          fs::ArrOp o = st.op;
          if (st.collapse) {
            o.kind = fs::HA_COLLAPSE;
          } else {
            o.kind = fs::HA_ACTIVE_ZERO;
            o.c0 = make_double2((a.flags & FS_NO_RENORM) ? 0.0 : 1.0, 0.0);
          }
          if ((rc = run_op(o, st.count))) return rc;
          break;
        }
      }
    }
    fs::hbm_finish_kernel<<<(W + 127) / 128, 128, 0, stream>>>(dp, a, H, batch0, W);
    p->launches++;
    FS_CUDA_TRY(cudaGetLastError());
    if (a.t_amps) {
      const int kst = (int)PL.final_live.size();
      fs::DevAxisMap m{};
      for (int b = 0; b < kst; b++) m.phys[b] = (int8_t)PL.final_live[b];
      const uint64_t sz = 1ull << kst;
      const uint64_t gx = std::max<uint64_t>(1, std::min<uint64_t>((sz + 255) / 256, 1024));
      fs::hbm_gather_kernel<<<dim3((unsigned)gx, (unsigned)nb), 256, 0, stream>>>(dp, a, H, batch0, (uint32_t)nb, kst, m,
                                                                                  a.t_amps);
      p->launches++;
      FS_CUDA_TRY(cudaGetLastError());
    }
  }
  return FS_OK;
}

int launch(fs_prog* p, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags, const fs_trace_in* tin,
           const fs_sample_out* out, const fs_trace_out* tout, cudaStream_t stream,
           const uint32_t* draw0 = nullptr) {
  if (shot0 % 32) return set_error(FS_ERR_ARG, "shot0 must be a multiple of 32");
  if (nshots == 0) return FS_OK;
  if (nshots > (uint64_t)0xFFFFFFFFull * 32) return set_error(FS_ERR_ARG, "too many shots for one call");
  if (!out || !out->accepted || !out->error) return set_error(FS_ERR_ARG, "missing output buffers");
  const fs::DevProg& dp = p->dp;
  if ((dp.U && !out->meas) || (dp.D && !out->det) || (dp.O && !out->obs))
    return set_error(FS_ERR_ARG, "missing output buffers");
  fs::RunArgs a{};
  a.seed = seed;
  a.shot0 = shot0;
  a.nshots = nshots;
  a.flags = flags;
  a.W = (uint32_t)((nshots + 31) / 32);
  a.ostride = a.W;
  a.meas = out->meas;
  a.det = out->det;
  a.obs = out->obs;
  a.accepted = out->accepted;
  a.error = out->error;
  a.status = out->status ? out->status : p->d_status;
  a.stop = dp.num_instrs;
  if (tin) {
    a.fault_modes = tin->fault_modes;
    a.forced = tin->forced;
    if (tin->stop >= 0 && tin->stop < dp.num_instrs) a.stop = tin->stop;
  }
  if (tout) {
    a.t_fx = tout->frame_x;
    a.t_fz = tout->frame_z;
    a.t_gamma = tout->gamma;
    a.t_amps = tout->amps;
    a.t_draws = tout->draws;
    a.t_rec = tout->records;
    if ((a.t_fx == nullptr) != (a.t_fz == nullptr)) return set_error(FS_ERR_ARG, "frame_x/frame_z must both be set");
    if (a.t_rec && dp.R) FS_CUDA_TRY(cudaMemsetAsync(a.t_rec, 0, nshots * (size_t)dp.R, stream));
  }
  if (tin && tin->ncheckpoints > 0) {  // checkpoint list (host) -> device, with amplitude offsets
    const int ncp = tin->ncheckpoints;
    if (!tin->checkpoints) return set_error(FS_ERR_ARG, "checkpoints is NULL");
    if (!tout || !tout->cp_valid || !tout->cp_frame_x || !tout->cp_frame_z || !tout->cp_gamma || !tout->cp_amps)
      return set_error(FS_ERR_ARG, "checkpoints need cp_valid, cp_frame_x/z, cp_gamma and cp_amps outputs");
    std::vector<int> at(tin->checkpoints, tin->checkpoints + ncp);
    std::vector<uint64_t> off(ncp);
    uint64_t o = 0;
    for (int j = 0; j < ncp; j++) {
      if (at[j] < 0 || at[j] > a.stop || (j && at[j] <= at[j - 1]))
        return set_error(FS_ERR_ARG, "checkpoints must be strictly ascending within [0, stop]");
      off[j] = o;
      o += nshots << (at[j] > 0 ? p->h_sched[at[j] - 1] : 0);
    }
    const size_t need = align_up(4 * (size_t)ncp, 16) + 8 * (size_t)ncp;
    if (need > p->cp_bytes) {
      cudaFree(p->d_cp);
      p->d_cp = nullptr;
      p->cp_bytes = 0;
      FS_CUDA_TRY(cudaMalloc(&p->d_cp, need));
      p->cp_bytes = need;
    }
    int* d_at = static_cast<int*>(p->d_cp);
    uint64_t* d_off = reinterpret_cast<uint64_t*>(static_cast<unsigned char*>(p->d_cp) + align_up(4 * (size_t)ncp, 16));
    FS_CUDA_TRY(cudaMemcpyAsync(d_at, at.data(), 4 * (size_t)ncp, cudaMemcpyHostToDevice, stream));
    FS_CUDA_TRY(cudaMemcpyAsync(d_off, off.data(), 8 * (size_t)ncp, cudaMemcpyHostToDevice, stream));
    FS_CUDA_TRY(cudaStreamSynchronize(stream));  // the host vectors go out of scope
    p->cp_list = at;
    p->cp_offs = off;
    a.ncp = ncp;
    a.cp_at = d_at;
    a.cp_off = d_off;
    a.cp_valid = tout->cp_valid;
    a.cp_fx = tout->cp_frame_x;
    a.cp_fz = tout->cp_frame_z;
    a.cp_gamma = tout->cp_gamma;
    a.cp_amps = tout->cp_amps;
    FS_CUDA_TRY(cudaMemsetAsync(a.cp_valid, 0, (size_t)ncp * nshots, stream));
  }
  a.arr_log2 = dp.k_max;
  a.draw0 = draw0;
  if (!out->status) FS_CUDA_TRY(cudaMemsetAsync(p->d_status, 0, sizeof(int), stream));
  if (wants_hbm(p, flags)) return launch_hbm(p, a, stream);
  const size_t W = a.W;
  a.prezeroed = 0;
  if (dp.has_psel) {  // halted warps may stop early: their remaining output words must read 0
    if (dp.U) FS_CUDA_TRY(cudaMemsetAsync(a.meas, 0, sizeof(uint32_t) * dp.U * W, stream));
    if (dp.D) FS_CUDA_TRY(cudaMemsetAsync(a.det, 0, sizeof(uint32_t) * dp.D * W, stream));
    a.prezeroed = 1;
  }
  const bool general = wants_general(p, flags, tin, tout);
  const bool trace_in = tin && (tin->fault_modes || tin->forced);
  const bool frame_free = !general && !trace_in && !(tout && tout->frame_x) && !(flags & FS_NO_JIT) &&
                          a.stop == dp.num_instrs && !p->env.no_affine;
  if (frame_free && ensure_aff(p) == FS_OK) return launch_aff(p, a, stream);
  if (!general && !trace_in && !(tout && tout->frame_x) && !(flags & FS_NO_JIT) && a.stop == dp.num_instrs) {
    int rc = ensure_jit(p);
    if (rc == FS_OK) {
      fsjit::Api& J = fsjit::api();
      const size_t smem = (size_t)4 * (p->jit_nslots + p->jit_stage) * 32 * sizeof(uint32_t);
      int occ = 1;
      J.cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->jit.fn, 128, smem);
      const size_t groups = (W + 127) / 128;
      const size_t grid = std::min<size_t>(groups, (size_t)p->num_sms * std::max(occ, 1));
      // fault lists (generator kernel, aux stream) pipelined with the frame kernel (main stream)
      // over NCH chunks of words: the list of chunk c+1 is generated while chunk c is simulated
      uint32_t *fent = nullptr, *bcount = nullptr, *ntot = nullptr;
      if ((rc = alloc_fault_lists(p, W, &fent, &bcount, &ntot))) return rc;
      if (!p->aux) {
        FS_CUDA_TRY(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking));
        for (int c = 0; c < kChunks + 1; c++) FS_CUDA_TRY(cudaEventCreateWithFlags(&p->ev[c], cudaEventDisableTiming));
      }
      int nch_req = 1;
      nch_req = p->env.jit_chunks;
      const int nch = W >= (size_t)nch_req * 4096 ? nch_req : 1;
      const size_t per = (W + nch - 1) / nch;
      FS_CUDA_TRY(cudaEventRecord(p->ev[kChunks], stream));
      FS_CUDA_TRY(cudaStreamWaitEvent(p->aux, p->ev[kChunks], 0));
      for (int c = 0; c < nch; c++) {
        const size_t w0 = c * per, nw = std::min(per, W - w0);
        if ((rc = run_fault_lists(p, a, w0, nw, fent, bcount, ntot, p->aux))) return rc;
        FS_CUDA_TRY(cudaEventRecord(p->ev[c], p->aux));
      }
      for (int c = 0; c < nch; c++) {
        const size_t w0 = c * per, nw = std::min(per, W - w0);
        FS_CUDA_TRY(cudaStreamWaitEvent(stream, p->ev[c], 0));
        fs::RunArgs ac = a;
        ac.W = (uint32_t)nw;
        ac.nshots = std::min<uint64_t>(a.nshots - w0 * 32, (uint64_t)nw * 32);
        ac.shot0 = a.shot0 + w0 * 32;
        ac.meas = a.meas ? a.meas + w0 : nullptr;
        ac.det = a.det ? a.det + w0 : nullptr;
        ac.obs = a.obs ? a.obs + w0 : nullptr;
        ac.accepted = a.accepted + w0;
        ac.error = a.error + w0;
        const size_t gc = std::min<size_t>((nw + 127) / 128, (size_t)p->num_sms * std::max(occ, 1));
        fs::DevProg dpv = dp;
        const uint16_t* ps = p->d_pslot;
        const uint32_t* fl = fent + w0;
        const uint32_t* fc = bcount + w0;
        const uint32_t* ft = ntot + w0;
        void* args[] = {&dpv, &ac, &ps, &fl, &fc, &ft};
        kt_begin(p, stream);
        int r = J.cuLaunchKernel(p->jit.fn, (unsigned)gc, 1, 1, 128, 1, 1, (unsigned)smem, stream, args, nullptr);
        kt_end(p, stream);
        p->launches++;
        if (r != 0) return set_error(FS_ERR_CUDA, "cuLaunchKernel(fs_jit_frame) failed: " + std::to_string(r));
      }
      (void)grid;
      return FS_OK;
    }
  }
  if (!general) {
    const int words_per_warp = 2 * dp.n + dp.num_slots + dp.O;
    const size_t smem = (size_t)fs::kFrameWarps * words_per_warp * 32 * sizeof(uint32_t);
    if (smem > kSmemBudget) return set_error(FS_ERR_ARG, "program too large for the frame engine");
    const bool trace = tin && (tin->fault_modes || tin->forced) || (tout && tout->frame_x);
    auto kern = trace ? fs::frame_kernel<true> : fs::frame_kernel<false>;
    FS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int threads = fs::kFrameWarps * 32;
    const size_t groups = (W + threads - 1) / threads;
    const int occ = occupancy_blocks(kern, threads, smem);
    const size_t grid = std::min<size_t>(groups, (size_t)p->num_sms * occ);
    kt_begin(p, stream);
    kern<<<(unsigned)grid, threads, smem, stream>>>(dp, a, words_per_warp);
    kt_end(p, stream);
    p->launches++;
    FS_CUDA_TRY(cudaGetLastError());
    return FS_OK;
  }
  // general engine
  const bool trace = (tin && (tin->fault_modes || tin->forced || tin->ncheckpoints > 0)) || tout;
  if (dp.has_psel && (!trace || (flags & FS_FORCE_SEGMENTED)) && a.stop == dp.num_instrs)
    return launch_segmented(p, a, stream);
  if (!(a.flags & (FS_RNG_SPLITMIX | FS_NO_RENORM | FS_NO_JIT | FS_FORCE_GENERAL)) && !trace &&
      a.stop == dp.num_instrs && gjit_supported(p) && ensure_gjit(p) == FS_OK) {
    uint32_t *fent = nullptr, *bcount = nullptr, *ntot = nullptr;
    int rc = alloc_fault_lists(p, a.W, &fent, &bcount, &ntot);
    if (rc) return rc;
    if (p->jit_nblocks && (rc = run_fault_lists(p, a, 0, a.W, fent, bcount, ntot, stream))) return rc;
    fsjit::Api& J = fsjit::api();
    if (p->gjit_occ == 0) {  // once per program
      int o1 = 1;
      J.cuOccupancyMaxActiveBlocksPerMultiprocessor(&o1, p->jit.fn, p->gjit_threads, p->gjit_smem);
      p->gjit_occ = std::max(o1, 1);
    }
    const int occ = p->gjit_occ;
    const int nw = p->gjit_threads / 32;
    const size_t blocks = (a.W + nw - 1) / nw;
    const size_t grid = std::min<size_t>(blocks, (size_t)p->num_sms * std::max(occ, 1));
    fs::DevProg dpv = dp;
    const uint16_t* ps = p->d_pslot;
    const uint32_t* fl = fent;
    const uint32_t* fc = bcount;
    const uint32_t* ft = ntot;
    void* args[] = {&dpv, &a, &ps, &fl, &fc, &ft};
    kt_begin(p, stream);
    int r = J.cuLaunchKernel(p->jit.fn, (unsigned)grid, 1, 1, p->gjit_threads, 1, 1, (unsigned)p->gjit_smem, stream,
                             args, nullptr);
    kt_end(p, stream);
    p->launches++;
    if (r != 0) return set_error(FS_ERR_CUDA, "cuLaunchKernel(fs_jit_general) failed: " + std::to_string(r));
    return FS_OK;
  }
  fs::SegArgs none{};
  return launch_general_kernel(p, a, none, false, dp.k_max, a.W, stream);
}

// popcount reduction of one sampling chunk into counts (sums over accepted shots)
__global__ void accumulate_kernel(const uint32_t* __restrict__ rows, int nrows, const uint32_t* __restrict__ acc,
                                  uint32_t W, int64_t* __restrict__ counts) {
  const int r = blockIdx.y;
  int64_t s = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x) {
    const uint32_t a = __ldg(acc + w);
    s += __popc((r < nrows ? __ldg(rows + (size_t)r * W + w) : 0xFFFFFFFFu) & a);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  __shared__ int64_t red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(counts + r), (unsigned long long)v);
  }
}

}  // namespace

extern "C" int fs_sample(fs_prog* p, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                         const fs_trace_in* tin, const fs_sample_out* out, const fs_trace_out* tout,
                         void* stream) {
  if (!p) return set_error(FS_ERR_ARG, "null program");
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  return launch(p, seed, shot0, nshots, flags, tin, out, tout, static_cast<cudaStream_t>(stream));
}


extern "C" int fs_sample_host(fs_prog* p, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                              const fs_trace_in* tin, const fs_sample_out* out, const fs_trace_out* tout) {
  if (!p || !out) return set_error(FS_ERR_ARG, "null argument");
  if (nshots == 0) return FS_OK;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  const fs::DevProg& dp = p->dp;
  const size_t W = (nshots + 31) / 32;
  int stop = dp.num_instrs;
  if (tin && tin->stop >= 0 && tin->stop < dp.num_instrs) stop = tin->stop;
  int k_stop = 0;
  if (stop > 0) k_stop = p->h_sched[stop - 1];
  const size_t n = (size_t)dp.n;
  // sizes
  size_t need = 0;
  auto acc = [&](size_t b) { need = align_up(need + b, 256); };
  acc(4 * W * dp.U); acc(4 * W * dp.D); acc(4 * W * dp.O); acc(4 * W); acc(4 * W); acc(4);
  const bool has_fm = tin && tin->fault_modes, has_fo = tin && tin->forced;
  if (has_fm) acc(2 * nshots * dp.E);
  if (has_fo) acc(nshots * dp.R);
  const int ncp = (tin && tin->ncheckpoints > 0 && tin->checkpoints) ? tin->ncheckpoints : 0;
  size_t cp_amp_elems = 0;  // complex elements of all checkpoint blocks
  for (int j = 0; j < ncp; j++) {
    const int c = tin->checkpoints[j];
    if (c < 0 || c > stop) return set_error(FS_ERR_ARG, "checkpoints must be strictly ascending within [0, stop]");
    cp_amp_elems += nshots << (c > 0 ? p->h_sched[c - 1] : 0);
  }
  if (tout) {
    if (tout->frame_x) { acc(nshots * n); acc(nshots * n); }
    if (tout->gamma) acc(16 * nshots);
    if (tout->amps) acc(16 * nshots * ((size_t)1 << k_stop));
    if (tout->draws) acc(4 * nshots);
    if (tout->records) acc(nshots * (size_t)dp.R);
    if (ncp) {
      acc(ncp * nshots); acc(ncp * nshots * n); acc(ncp * nshots * n); acc(16 * ncp * nshots);
      acc(16 * cp_amp_elems);
    }
  }
  if (need > p->stage_bytes) {
    cudaFree(p->stage);
    p->stage = nullptr;
    p->stage_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->stage, need));
    p->stage_bytes = need;
  }
  Stage st;
  st.base = static_cast<unsigned char*>(p->stage);
  fs_sample_out dout{};
  dout.meas = st.take<uint32_t>(W * dp.U);
  dout.det = st.take<uint32_t>(W * dp.D);
  dout.obs = st.take<uint32_t>(W * dp.O);
  dout.accepted = st.take<uint32_t>(W);
  dout.error = st.take<uint32_t>(W);
  dout.status = st.take<int32_t>(1);
  cudaStream_t s = 0;
  FS_CUDA_TRY(cudaMemsetAsync(dout.status, 0, 4, s));
  fs_trace_in dtin{};
  fs_trace_in* ptin = nullptr;
  if (tin) {
    dtin.stop = tin->stop;
    dtin.ncheckpoints = tin->ncheckpoints;  // host list, read by launch()
    dtin.checkpoints = tin->checkpoints;
    if (has_fm) {
      int16_t* d = st.take<int16_t>(nshots * dp.E);
      FS_CUDA_TRY(cudaMemcpyAsync(d, tin->fault_modes, 2 * nshots * dp.E, cudaMemcpyHostToDevice, s));
      dtin.fault_modes = d;
    }
    if (has_fo) {
      int8_t* d = st.take<int8_t>(nshots * dp.R);
      FS_CUDA_TRY(cudaMemcpyAsync(d, tin->forced, nshots * dp.R, cudaMemcpyHostToDevice, s));
      dtin.forced = d;
    }
    ptin = &dtin;
  }
  fs_trace_out dtout{};
  fs_trace_out* ptout = nullptr;
  if (tout) {
    if (tout->frame_x) { dtout.frame_x = st.take<uint8_t>(nshots * n); dtout.frame_z = st.take<uint8_t>(nshots * n); }
    if (tout->gamma) dtout.gamma = st.take<double>(2 * nshots);
    if (tout->amps) dtout.amps = st.take<double>(2 * nshots * ((size_t)1 << k_stop));
    if (tout->draws) dtout.draws = st.take<uint32_t>(nshots);
    if (tout->records) dtout.records = st.take<uint8_t>(nshots * (size_t)dp.R);
    if (ncp) {
      dtout.cp_valid = st.take<uint8_t>(ncp * nshots);
      dtout.cp_frame_x = st.take<uint8_t>(ncp * nshots * n);
      dtout.cp_frame_z = st.take<uint8_t>(ncp * nshots * n);
      dtout.cp_gamma = st.take<double>(2 * ncp * nshots);
      dtout.cp_amps = st.take<double>(2 * cp_amp_elems);
    }
    ptout = &dtout;
  }
  int rc = launch(p, seed, shot0, nshots, flags, ptin, &dout, ptout, s);
  if (rc != FS_OK) return rc;
  if (dp.U) FS_CUDA_TRY(cudaMemcpyAsync(out->meas, dout.meas, 4 * W * dp.U, cudaMemcpyDeviceToHost, s));
  if (dp.D) FS_CUDA_TRY(cudaMemcpyAsync(out->det, dout.det, 4 * W * dp.D, cudaMemcpyDeviceToHost, s));
  if (dp.O) FS_CUDA_TRY(cudaMemcpyAsync(out->obs, dout.obs, 4 * W * dp.O, cudaMemcpyDeviceToHost, s));
  FS_CUDA_TRY(cudaMemcpyAsync(out->accepted, dout.accepted, 4 * W, cudaMemcpyDeviceToHost, s));
  FS_CUDA_TRY(cudaMemcpyAsync(out->error, dout.error, 4 * W, cudaMemcpyDeviceToHost, s));
  int status = 0;
  FS_CUDA_TRY(cudaMemcpyAsync(&status, dout.status, 4, cudaMemcpyDeviceToHost, s));
  if (tout) {
    if (tout->frame_x) {
      FS_CUDA_TRY(cudaMemcpyAsync(tout->frame_x, dtout.frame_x, nshots * n, cudaMemcpyDeviceToHost, s));
      FS_CUDA_TRY(cudaMemcpyAsync(tout->frame_z, dtout.frame_z, nshots * n, cudaMemcpyDeviceToHost, s));
    }
    if (tout->gamma) FS_CUDA_TRY(cudaMemcpyAsync(tout->gamma, dtout.gamma, 16 * nshots, cudaMemcpyDeviceToHost, s));
    if (tout->amps)
      FS_CUDA_TRY(cudaMemcpyAsync(tout->amps, dtout.amps, 16 * nshots * ((size_t)1 << k_stop), cudaMemcpyDeviceToHost, s));
    if (tout->draws) FS_CUDA_TRY(cudaMemcpyAsync(tout->draws, dtout.draws, 4 * nshots, cudaMemcpyDeviceToHost, s));
    if (tout->records && dp.R)
      FS_CUDA_TRY(cudaMemcpyAsync(tout->records, dtout.records, nshots * (size_t)dp.R, cudaMemcpyDeviceToHost, s));
    if (ncp) {
      if (tout->cp_valid) FS_CUDA_TRY(cudaMemcpyAsync(tout->cp_valid, dtout.cp_valid, ncp * nshots, cudaMemcpyDeviceToHost, s));
      if (tout->cp_frame_x) FS_CUDA_TRY(cudaMemcpyAsync(tout->cp_frame_x, dtout.cp_frame_x, ncp * nshots * n, cudaMemcpyDeviceToHost, s));
      if (tout->cp_frame_z) FS_CUDA_TRY(cudaMemcpyAsync(tout->cp_frame_z, dtout.cp_frame_z, ncp * nshots * n, cudaMemcpyDeviceToHost, s));
      if (tout->cp_gamma) FS_CUDA_TRY(cudaMemcpyAsync(tout->cp_gamma, dtout.cp_gamma, 16 * ncp * nshots, cudaMemcpyDeviceToHost, s));
      if (tout->cp_amps) FS_CUDA_TRY(cudaMemcpyAsync(tout->cp_amps, dtout.cp_amps, 16 * cp_amp_elems, cudaMemcpyDeviceToHost, s));
    }
  }
  FS_CUDA_TRY(cudaStreamSynchronize(s));
  if (out->status) *out->status = status;
  if (status) {
    g_last_error = status == FS_ERR_SHOT_NAN ? "NaN amplitude encountered at an active measurement"
                                             : "forced outcome has probability below BRANCH_FLOOR";
  }
  return status;
}

namespace {
// device status of a whole call -> host (synchronizes the stream); sets the error text
int finish_status(const int32_t* status_d, cudaStream_t stream) {
  int32_t status = 0;
  FS_CUDA_TRY(cudaMemcpyAsync(&status, status_d, 4, cudaMemcpyDeviceToHost, stream));
  FS_CUDA_TRY(cudaStreamSynchronize(stream));
  if (status == FS_ERR_SHOT_NAN) g_last_error = "NaN amplitude encountered at an active measurement";
  else if (status) g_last_error = "forced outcome has probability below BRANCH_FLOOR";
  return status;
}
}  // namespace

extern "C" int fs_accumulate(fs_prog* p, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                             int64_t* counts, void* stream_) {
  if (!p || !counts) return set_error(FS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const fs::DevProg& dp = p->dp;
  const int nrows = dp.U + dp.D + dp.O;
  FS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (nrows + 1), stream));
  const uint64_t chunk = (uint64_t)1 << 22;
  const size_t Wc = chunk / 32;
  const size_t need = align_up(4 * Wc * (nrows + 2) + 256, 256);
  if (need > p->stage_bytes) {
    cudaFree(p->stage);
    p->stage = nullptr;
    p->stage_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->stage, need));
    p->stage_bytes = need;
  }
  // shots that raised (NaN / impossible forced outcome) are not silently counted as rejected:
  // the call returns their status like fs_sample (the reference propagates ShotError)
  int32_t* status_d = reinterpret_cast<int32_t*>(static_cast<unsigned char*>(p->stage) + 4 * Wc * (nrows + 2));
  FS_CUDA_TRY(cudaMemsetAsync(status_d, 0, 4, stream));
  for (uint64_t s0 = 0; s0 < nshots; s0 += chunk) {
    const uint64_t ns = std::min<uint64_t>(chunk, nshots - s0);
    const uint32_t W = (uint32_t)((ns + 31) / 32);
    Stage st;
    st.base = static_cast<unsigned char*>(p->stage);
    uint32_t* rows = st.take<uint32_t>((size_t)W * (nrows + 2));
    fs_sample_out o{};
    o.meas = rows;
    o.det = rows + (size_t)W * dp.U;
    o.obs = rows + (size_t)W * (dp.U + dp.D);
    o.accepted = rows + (size_t)W * nrows;
    o.error = rows + (size_t)W * (nrows + 1);
    o.status = status_d;  // accumulates (atomicMax) over every chunk of the call
    int rc = launch(p, seed, shot0 + s0, ns, flags, nullptr, &o, nullptr, stream);
    if (rc != FS_OK) return rc;
    dim3 grid(std::min<uint32_t>((W + 255) / 256, 64), nrows + 1);
    accumulate_kernel<<<grid, 256, 0, stream>>>(rows, nrows, o.accepted, W, counts);
    p->launches++;
    FS_CUDA_TRY(cudaGetLastError());
  }
  return finish_status(status_d, stream);
}

// ------------------------------------------------------------------ output formats (cli.py)
namespace {
int fmt_nbits(const fs_prog* p) { return p->dp.U + p->dp.D + p->dp.O; }
uint64_t dec_digits_h(uint64_t v) {
  uint64_t d = 1;
  while (v >= 10) { v /= 10; d++; }
  return d;
}
}  // namespace

extern "C" uint64_t fs_format_bound(const fs_prog* p, uint64_t nshots, int format, uint64_t index0,
                                    const char* weight_text) {
  if (!p) return 0;
  const uint64_t nb = (uint64_t)fmt_nbits(p);
  if (format == FS_FMT_BIN) return nshots * ((nb + 7) / 8);
  if (format == FS_FMT_CSV) {
    const uint64_t wl = weight_text ? std::strlen(weight_text) : 1;
    return nshots * (dec_digits_h(index0 + nshots) + 2 + wl + nb + 1);
  }
  return nshots * (nb + 1 + 9);
}

extern "C" int fs_format(fs_prog* p, const fs_sample_out* words, uint64_t nshots, int format, int keep_rejected,
                         uint64_t index0, const char* weight_text, uint8_t* dst, uint64_t cap, uint64_t* nbytes,
                         uint64_t* nkept, void* stream_) {
  if (!p || !words || !dst || !nbytes) return set_error(FS_ERR_ARG, "null argument");
  if (format < FS_FMT_01 || format > FS_FMT_CSV) return set_error(FS_ERR_ARG, "unknown format");
  *nbytes = 0;
  if (nkept) *nkept = 0;
  if (nshots == 0) return FS_OK;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const fs::DevProg& dp = p->dp;
  const char* wt = weight_text ? weight_text : "1";
  const int wlen = (int)std::strlen(wt);
  if (wlen > 64) return set_error(FS_ERR_ARG, "weight text longer than 64 characters");
  // scratch: kept u32, rank u32, len u64, off u64, weight text, scan temp
  size_t t1 = 0, t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, (uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)nshots, stream);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)nshots, stream);
  const size_t temp = std::max(t1, t2);
  const size_t need = align_up(4 * nshots, 256) * 2 + align_up(8 * nshots, 256) * 2 + 256 + align_up(temp, 256);
  if (need > p->fmt_bytes) {
    cudaFree(p->fmt);
    p->fmt = nullptr;
    p->fmt_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->fmt, need));
    p->fmt_bytes = need;
  }
  Stage st;
  st.base = static_cast<unsigned char*>(p->fmt);
  uint32_t* kept = st.take<uint32_t>(nshots);
  uint32_t* rank = st.take<uint32_t>(nshots);
  uint64_t* len = st.take<uint64_t>(nshots);
  uint64_t* off = st.take<uint64_t>(nshots);
  char* dw = st.take<char>(256);
  void* tmp = st.take<unsigned char>(temp);
  FS_CUDA_TRY(cudaMemcpyAsync(dw, wt, wlen + 1, cudaMemcpyHostToDevice, stream));
  fs::FmtArgs F{};
  F.meas = words->meas;
  F.det = words->det;
  F.obs = words->obs;
  F.accepted = words->accepted;
  F.n = nshots;
  F.W = (uint32_t)((nshots + 31) / 32);
  F.U = dp.U;
  F.D = dp.D;
  F.O = dp.O;
  F.format = format;
  F.keep_rejected = keep_rejected ? 1 : 0;
  F.index0 = index0;
  F.weight = dw;
  F.wlen = wlen;
  const unsigned g = (unsigned)((nshots + 255) / 256);
  fs::fmt_kept_kernel<<<g, 256, 0, stream>>>(F, kept);
  size_t tb = temp;
  FS_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, kept, rank, (int64_t)nshots, stream));
  fs::fmt_len_kernel<<<g, 256, 0, stream>>>(F, kept, rank, len);
  tb = temp;
  FS_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, len, off, (int64_t)nshots, stream));
  uint64_t last[2] = {0, 0};
  uint32_t lk2[2] = {0, 0};
  FS_CUDA_TRY(cudaMemcpyAsync(&last[0], off + nshots - 1, 8, cudaMemcpyDeviceToHost, stream));
  FS_CUDA_TRY(cudaMemcpyAsync(&last[1], len + nshots - 1, 8, cudaMemcpyDeviceToHost, stream));
  FS_CUDA_TRY(cudaMemcpyAsync(&lk2[0], rank + nshots - 1, 4, cudaMemcpyDeviceToHost, stream));
  FS_CUDA_TRY(cudaMemcpyAsync(&lk2[1], kept + nshots - 1, 4, cudaMemcpyDeviceToHost, stream));
  FS_CUDA_TRY(cudaStreamSynchronize(stream));
  const uint64_t total = last[0] + last[1];
  if (total > cap) return set_error(FS_ERR_ARG, "format destination too small (see fs_format_bound)");
  fs::fmt_write_kernel<<<g, 256, 0, stream>>>(F, kept, rank, off, dst);
  p->launches += 4;
  FS_CUDA_TRY(cudaGetLastError());
  *nbytes = total;
  if (nkept) *nkept = (uint64_t)lk2[0] + lk2[1];
  return FS_OK;
}

// ------------------------------------------------------------------ stratified sampling
namespace {
// suffix[i][m] = Pr[m faults among sites i..E-1] for m <= w, built exactly like StratumSpec
// (runtime.py:898-908): nxt[m] = prev[m] * (1 - p) + prev[m - 1] * p in that order
int stratum_prepare(fs_prog* p, uint32_t w) {
  const int E = p->dp.E;
  if ((int64_t)w > E)
    return set_error(FS_ERR_ARG, "stratum fault count " + std::to_string(w) + " exceeds " + std::to_string(E) + " sites");
  if (p->strat_w == (int)w && p->d_strat) return FS_OK;
  const size_t w1 = (size_t)w + 1;
  std::vector<double> T((size_t)(E + 1) * w1, 0.0);
  T[(size_t)E * w1] = 1.0;
  for (int i = E - 1; i >= 0; i--) {
    const double pr = p->h_site_prob[i];
    const double omp = 1.0 - pr;
    const double* prev = T.data() + (size_t)(i + 1) * w1;
    double* nxt = T.data() + (size_t)i * w1;
    for (size_t m = 0; m < w1; m++) {
      volatile double a = prev[m] * omp;  // volatile: no contraction into an FMA
      double v = a;
      if (m) {
        volatile double b = prev[m - 1] * pr;
        v = a + b;
      }
      nxt[m] = v;
    }
  }
  cudaFree(p->d_strat);
  p->d_strat = nullptr;
  FS_CUDA_TRY(cudaMalloc(&p->d_strat, sizeof(double) * T.size()));
  FS_CUDA_TRY(cudaMemcpy(p->d_strat, T.data(), sizeof(double) * T.size(), cudaMemcpyHostToDevice));
  p->strat_w = (int)w;
  p->strat_weight = T[w];
  return FS_OK;
}

// stratified shots [shot0, shot0 + nshots) into device outputs (row stride ceil(nshots / 32));
// caller holds p->mu
int sample_stratum_impl(fs_prog* p, uint32_t w, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                        const fs_sample_out* out, cudaStream_t stream) {
  if (shot0 % 32) return set_error(FS_ERR_ARG, "shot0 must be a multiple of 32");
  if (int rc = stratum_prepare(p, w)) return rc;
  const fs::DevProg& dp = p->dp;
  const size_t E = (size_t)std::max(dp.E, 1);
  const size_t W = (nshots + 31) / 32;
  const int rows = dp.U + dp.D + dp.O + 2;
  uint64_t chunk = std::max<uint64_t>(32, ((uint64_t)1 << 30) / (2 * E) / 32 * 32);
  if (p->env.stratum_chunk) chunk = p->env.stratum_chunk;  // tests
  chunk = std::min<uint64_t>(chunk, (nshots + 31) / 32 * 32);
  const size_t Wc = chunk / 32;
  const size_t need = align_up(2 * E * chunk, 256) + align_up(4 * chunk, 256) + align_up(4 * Wc * rows, 256) + 256;
  if (need > p->strat_bytes) {
    cudaFree(p->strat_buf);
    p->strat_buf = nullptr;
    p->strat_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->strat_buf, need));
    p->strat_bytes = need;
  }
  Stage st;
  st.base = static_cast<unsigned char*>(p->strat_buf);
  int16_t* modes = st.take<int16_t>(E * chunk);
  uint32_t* draw0 = st.take<uint32_t>(chunk);
  uint32_t* crow = st.take<uint32_t>(Wc * rows);
  const bool splitmix = flags & FS_RNG_SPLITMIX;
  for (uint64_t c0 = 0; c0 < nshots; c0 += chunk) {
    const uint64_t nc = std::min<uint64_t>(chunk, nshots - c0);
    const size_t wc = (nc + 31) / 32;
    const uint64_t cells = nc * (uint64_t)dp.E;
    if (cells) {
      fs::fill_modes_kernel<<<(unsigned)((cells / 8 + 1 + 255) / 256), 256, 0, stream>>>(modes, cells);
      p->launches++;
    }
    const unsigned g = (unsigned)((nc + 127) / 128);
    if (splitmix) fs::stratum_kernel<true><<<g, 128, 0, stream>>>(dp, p->d_strat, (int)w, seed, shot0 + c0, nc, modes, draw0);
    else fs::stratum_kernel<false><<<g, 128, 0, stream>>>(dp, p->d_strat, (int)w, seed, shot0 + c0, nc, modes, draw0);
    p->launches++;
    FS_CUDA_TRY(cudaGetLastError());
    fs_trace_in tin{};
    tin.fault_modes = dp.E ? modes : nullptr;
    tin.forced = nullptr;
    tin.stop = -1;
    const bool whole = nc == nshots;
    fs_sample_out o{};
    if (whole) {
      o = *out;
    } else {
      o.meas = crow;
      o.det = crow + wc * dp.U;
      o.obs = crow + wc * (dp.U + dp.D);
      o.accepted = crow + wc * (dp.U + dp.D + dp.O);
      o.error = o.accepted + wc;
      o.status = out->status;
    }
    int rc = launch(p, seed, shot0 + c0, nc, flags, &tin, &o, nullptr, stream, splitmix ? draw0 : nullptr);
    if (rc != FS_OK) return rc;
    if (!whole) {  // place the chunk's words at word offset c0 / 32 of every output row
      const size_t w0 = c0 / 32;
      auto put = [&](uint32_t* dst, const uint32_t* src, int nrow) -> int {
        if (!nrow || !dst) return FS_OK;
        FS_CUDA_TRY(cudaMemcpy2DAsync(dst + w0, 4 * W, src, 4 * wc, 4 * wc, nrow, cudaMemcpyDeviceToDevice, stream));
        return FS_OK;
      };
      if ((rc = put(out->meas, o.meas, dp.U)) || (rc = put(out->det, o.det, dp.D)) || (rc = put(out->obs, o.obs, dp.O)) ||
          (rc = put(out->accepted, o.accepted, 1)) || (rc = put(out->error, o.error, 1)))
        return rc;
    }
  }
  return FS_OK;
}
}  // namespace

extern "C" int fs_stratum_weight(fs_prog* p, uint32_t w, double* weight) {
  if (!p || !weight) return set_error(FS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  if (int rc = stratum_prepare(p, w)) return rc;
  *weight = p->strat_weight;
  return FS_OK;
}

extern "C" int fs_sample_stratum(fs_prog* p, uint32_t w, uint64_t seed, uint64_t shot0, uint64_t nshots,
                                 uint32_t flags, const fs_sample_out* out, void* stream) {
  if (!p || !out) return set_error(FS_ERR_ARG, "null argument");
  if (nshots == 0) return FS_OK;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  return sample_stratum_impl(p, w, seed, shot0, nshots, flags, out, static_cast<cudaStream_t>(stream));
}

extern "C" int fs_sample_stratum_host(fs_prog* p, uint32_t w, uint64_t seed, uint64_t shot0, uint64_t nshots,
                                      uint32_t flags, const fs_sample_out* out) {
  if (!p || !out) return set_error(FS_ERR_ARG, "null argument");
  if (nshots == 0) return FS_OK;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  const fs::DevProg& dp = p->dp;
  const size_t W = (nshots + 31) / 32;
  const size_t rows = (size_t)dp.U + dp.D + dp.O + 2;
  const size_t need = align_up(4 * W * rows + 64, 256);
  if (need > p->stage_bytes) {
    cudaFree(p->stage);
    p->stage = nullptr;
    p->stage_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->stage, need));
    p->stage_bytes = need;
  }
  uint32_t* r = static_cast<uint32_t*>(p->stage);
  fs_sample_out d{};
  d.meas = r;
  d.det = r + W * dp.U;
  d.obs = r + W * (dp.U + dp.D);
  d.accepted = r + W * (dp.U + dp.D + dp.O);
  d.error = d.accepted + W;
  d.status = reinterpret_cast<int32_t*>(d.error + W);
  cudaStream_t s = 0;
  FS_CUDA_TRY(cudaMemsetAsync(d.status, 0, 4, s));
  int rc = sample_stratum_impl(p, w, seed, shot0, nshots, flags, &d, s);
  if (rc != FS_OK) return rc;
  if (dp.U) FS_CUDA_TRY(cudaMemcpyAsync(out->meas, d.meas, 4 * W * dp.U, cudaMemcpyDeviceToHost, s));
  if (dp.D) FS_CUDA_TRY(cudaMemcpyAsync(out->det, d.det, 4 * W * dp.D, cudaMemcpyDeviceToHost, s));
  if (dp.O) FS_CUDA_TRY(cudaMemcpyAsync(out->obs, d.obs, 4 * W * dp.O, cudaMemcpyDeviceToHost, s));
  FS_CUDA_TRY(cudaMemcpyAsync(out->accepted, d.accepted, 4 * W, cudaMemcpyDeviceToHost, s));
  FS_CUDA_TRY(cudaMemcpyAsync(out->error, d.error, 4 * W, cudaMemcpyDeviceToHost, s));
  int status = 0;
  FS_CUDA_TRY(cudaMemcpyAsync(&status, d.status, 4, cudaMemcpyDeviceToHost, s));
  FS_CUDA_TRY(cudaStreamSynchronize(s));
  if (out->status) *out->status = status;
  if (status) {
    g_last_error = status == FS_ERR_SHOT_NAN ? "NaN amplitude encountered at an active measurement"
                                             : "forced outcome has probability below BRANCH_FLOOR";
  }
  return status;
}

extern "C" int fs_accumulate_stratum(fs_prog* p, uint32_t w, uint64_t seed, uint64_t shot0, uint64_t nshots,
                                     uint32_t flags, int64_t* counts, void* stream_) {
  if (!p || !counts) return set_error(FS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const fs::DevProg& dp = p->dp;
  const int nrows = dp.U + dp.D + dp.O;
  FS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (nrows + 1), stream));
  const uint64_t chunk = (uint64_t)1 << 22;
  const size_t Wc = chunk / 32;
  const size_t need = align_up(4 * Wc * (nrows + 2) + 256, 256);
  if (need > p->stage_bytes) {
    cudaFree(p->stage);
    p->stage = nullptr;
    p->stage_bytes = 0;
    FS_CUDA_TRY(cudaMalloc(&p->stage, need));
    p->stage_bytes = need;
  }
  // shots that raised (NaN / impossible forced outcome) are not silently counted as rejected:
  // the call returns their status like fs_sample (the reference propagates ShotError)
  int32_t* status_d = reinterpret_cast<int32_t*>(static_cast<unsigned char*>(p->stage) + 4 * Wc * (nrows + 2));
  FS_CUDA_TRY(cudaMemsetAsync(status_d, 0, 4, stream));
  for (uint64_t s0 = 0; s0 < nshots; s0 += chunk) {
    const uint64_t ns = std::min<uint64_t>(chunk, nshots - s0);
    const uint32_t W = (uint32_t)((ns + 31) / 32);
    uint32_t* rows = static_cast<uint32_t*>(p->stage);
    fs_sample_out o{};
    o.meas = rows;
    o.det = rows + (size_t)W * dp.U;
    o.obs = rows + (size_t)W * (dp.U + dp.D);
    o.accepted = rows + (size_t)W * nrows;
    o.error = rows + (size_t)W * (nrows + 1);
    o.status = status_d;
    int rc = sample_stratum_impl(p, w, seed, shot0 + s0, ns, flags, &o, stream);
    if (rc != FS_OK) return rc;
    dim3 grid(std::min<uint32_t>((W + 255) / 256, 64), nrows + 1);
    accumulate_kernel<<<grid, 256, 0, stream>>>(rows, nrows, o.accepted, W, counts);
    p->launches++;
    FS_CUDA_TRY(cudaGetLastError());
  }
  return finish_status(status_d, stream);
}

// ------------------------------------------------------------------ expectation probe
namespace {
constexpr int kProbeBlocks = 296;
// <a| i^y (-1)^{popc(idx & zm)} |a[idx ^ xm]> terms and |a|^2, per block (fixed order within a
// block), finished on the host in block order (runtime.py:951-989, one traversal)
__global__ void probe_kernel(const double2* __restrict__ a, uint64_t size, uint64_t xm, uint64_t zm, int y,
                             double* __restrict__ part) {
  double re = 0.0, nn = 0.0;
  const double2 iy = (y & 3) == 0 ? make_double2(1, 0) : (y & 3) == 1 ? make_double2(0, 1)
                   : (y & 3) == 2 ? make_double2(-1, 0) : make_double2(0, -1);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += (uint64_t)gridDim.x * blockDim.x) {
    const double2 ai = a[i], aj = a[i ^ xm];
    double2 t = fs::cmul(iy, ai);
    if (__popcll(i & zm) & 1) t = make_double2(-t.x, -t.y);
    re = __dadd_rn(re, __dadd_rn(__dmul_rn(aj.x, t.x), __dmul_rn(aj.y, t.y)));  // Re(conj(aj) * t)
    nn = __dadd_rn(nn, fs::cnorm2(ai));
  }
  __shared__ double s1[256], s2[256];
  s1[threadIdx.x] = re;
  s2[threadIdx.x] = nn;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if ((int)threadIdx.x < w) {
      s1[threadIdx.x] = __dadd_rn(s1[threadIdx.x], s1[threadIdx.x + w]);
      s2[threadIdx.x] = __dadd_rn(s2[threadIdx.x], s2[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s1[0];
    part[2 * blockIdx.x + 1] = s2[0];
  }
}
}  // namespace

extern "C" int fs_probe(const double* amps, int32_t k, uint64_t xm, uint64_t zm, int32_t ycount, double* out,
                        void* stream_) {
  if (!amps || !out || k < 0 || k > 40) return set_error(FS_ERR_ARG, "bad probe arguments");
  const uint64_t size = 1ull << k;
  if ((xm | zm) >> k) return set_error(FS_ERR_ARG, "probe masks outside the active array");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  static thread_local double* part = nullptr;
  if (!part) FS_CUDA_TRY(cudaMalloc(&part, sizeof(double) * 2 * kProbeBlocks));
  const unsigned g = (unsigned)std::min<uint64_t>(kProbeBlocks, (size + 255) / 256);
  probe_kernel<<<g, 256, 0, stream>>>(reinterpret_cast<const double2*>(amps), size, xm, zm, ycount, part);
  FS_CUDA_TRY(cudaGetLastError());
  std::vector<double> h(2 * g);
  FS_CUDA_TRY(cudaMemcpyAsync(h.data(), part, sizeof(double) * 2 * g, cudaMemcpyDeviceToHost, stream));
  FS_CUDA_TRY(cudaStreamSynchronize(stream));
  double re = 0.0, nn = 0.0;
  for (unsigned b = 0; b < g; b++) { re += h[2 * b]; nn += h[2 * b + 1]; }
  out[0] = re;
  out[1] = nn;
  return FS_OK;
}
