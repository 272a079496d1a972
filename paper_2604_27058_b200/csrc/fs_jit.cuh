// fs_jit.cuh -- host side of the program-specialised frame kernel (NVRTC + CUDA driver API).
//
// For a frame-only program (k_max = 0) sampled with the Philox stream, fs_program_create's
// first fs_sample call generates a CUDA kernel in which every bytecode instruction is unrolled
// with constant operands, compiles it for sm_100a with NVRTC and loads it with the driver API.
// Differences from the interpreter (fs_frame.cuh): no instruction fetch/decode, H / SWAP and
// the x<->z swap of MeasDormantRandom are renamings resolved by the generator (zero runtime
// cost), record slots / observables are registers, frame slots are constant smem offsets that
// the compiler keeps in registers between noise blocks.  Results are bit-identical to the
// interpreter (tests/test_gpu_parity.py::test_gpu_jit_equals_interpreter).
//
// libnvrtc and libcuda are loaded with dlopen so the library itself has no link-time CUDA
// driver dependency (it still loads on a CPU-only host; every entry point then fails loudly).
#pragma once
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <sstream>
#include <string>
#include <vector>

namespace fsjit {

constexpr int kJitStage = 64;  // staged fault entries per word (more -> in-place generation)

typedef int CUresult;
typedef void* CUmodule;
typedef void* CUfunction;
typedef void* CUstream;
typedef void* CUcontext;

struct Api {
  bool ok = false;
  std::string why;
  // nvrtc
  int (*nvrtcCreateProgram)(void**, const char*, const char*, int, const char* const*, const char* const*);
  int (*nvrtcCompileProgram)(void*, int, const char* const*);
  int (*nvrtcGetProgramLogSize)(void*, size_t*);
  int (*nvrtcGetProgramLog)(void*, char*);
  int (*nvrtcGetCUBINSize)(void*, size_t*);
  int (*nvrtcGetCUBIN)(void*, char*);
  int (*nvrtcDestroyProgram)(void**);
  // driver
  CUresult (*cuModuleLoadData)(CUmodule*, const void*);
  CUresult (*cuModuleGetFunction)(CUfunction*, CUmodule, const char*);
  CUresult (*cuModuleUnload)(CUmodule);
  CUresult (*cuFuncSetAttribute)(CUfunction, int, int);
  CUresult (*cuLaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void**, void**);
  CUresult (*cuOccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t);
  CUresult (*cuCtxGetCurrent)(CUcontext*);
};

inline void* try_open(const std::vector<std::string>& names) {
  for (auto& n : names) {
    void* h = dlopen(n.c_str(), RTLD_NOW | RTLD_GLOBAL);
    if (h) return h;
  }
  return nullptr;
}

inline std::string self_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&try_open), &info) && info.dli_fname) {
    std::string p(info.dli_fname);
    auto s = p.rfind('/');
    if (s != std::string::npos) return p.substr(0, s);
  }
  return ".";
}

inline Api load_api() {
  Api a;
  void* nv = try_open({"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"});
  void* cu = try_open({"libcuda.so.1", "libcuda.so"});
  if (!nv || !cu) {
    a.why = !nv ? "libnvrtc.so.12 not found" : "libcuda.so.1 not found";
    return a;
  }
#define LOAD(h, name)                                                      \
  a.name = reinterpret_cast<decltype(a.name)>(dlsym(h, #name));            \
  if (!a.name) { a.why = std::string("missing symbol ") + #name; return a; }
  LOAD(nv, nvrtcCreateProgram);
  LOAD(nv, nvrtcCompileProgram);
  LOAD(nv, nvrtcGetProgramLogSize);
  LOAD(nv, nvrtcGetProgramLog);
  LOAD(nv, nvrtcGetCUBINSize);
  LOAD(nv, nvrtcGetCUBIN);
  LOAD(nv, nvrtcDestroyProgram);
  LOAD(cu, cuModuleLoadData);
  LOAD(cu, cuModuleGetFunction);
  LOAD(cu, cuModuleUnload);
  LOAD(cu, cuFuncSetAttribute);
  LOAD(cu, cuLaunchKernel);
  LOAD(cu, cuOccupancyMaxActiveBlocksPerMultiprocessor);
  LOAD(cu, cuCtxGetCurrent);
#undef LOAD
  a.ok = true;
  return a;
}

// loaded once, thread-safely (C++11 magic static); callers check .ok before any driver call
inline Api& api() {
  static Api a = load_api();
  return a;
}

struct FrameKernelSource {
  std::string src;
  std::vector<uint16_t> pslot;  // per Pauli entry: physical slot under the renaming at its block
  int nslots = 0;               // physical frame slots (2n)
  int stage = kJitStage;        // staged fault entries per word (smem rows per warp)
  std::vector<int32_t> site_block;  // NoiseBlock ordinal of every site
  int nblocks = 0;
  std::vector<int32_t> block_hi, block_cap, row_off;  // flip rows per NoiseBlock
  int rows = 0, capmax = 0;
};

// Generate the specialised frame kernel for a frame-only program.
inline FrameKernelSource gen_frame_kernel(const fs_prog_desc& d, const std::vector<int32_t>& ins_all,
                                          const std::vector<uint32_t>& gates, const std::vector<uint32_t>& paulis,
                                          const std::vector<int32_t>& reclists, const std::vector<int32_t>& record_out,
                                          const std::vector<int32_t>& bit_slot, const std::vector<int32_t>& plans,
                                          const std::vector<int32_t>& case_pauli_off,
                                          const std::vector<int32_t>& site_case_off,
                                          const std::vector<double>& site_prob) {
  FrameKernelSource K;
  const int n = d.n;
  K.nslots = 2 * n;
  // fault staging depth: shrink it (not below 40) when that fits a third 4-warp block per SM
  // (3 x (smem + 1 KiB reserve) <= 228 KiB); words with more faults generate in place
  {
    const int fit = 76800 / (4 * 32 * 4) - K.nslots;
    if (fit >= 40 && fit < kJitStage) K.stage = fit;
    if (const char* e = getenv("FS_JIT_STAGE")) K.stage = std::max(8, std::min(kJitStage, atoi(e)));
  }
  K.site_block.assign(d.num_sites + 1, 0);
  for (int i = 0, b = 0; i < d.num_instrs; i++)
    if (FS_OPCODE(ins_all[(size_t)i * FS_INS_WORDS]) == FS_OP_NOISE) {
      const int lo = ins_all[(size_t)i * FS_INS_WORDS + 1], hi = ins_all[(size_t)i * FS_INS_WORDS + 2];
      double mu = 0.0;  // expected flips per 32-shot word in this block
      for (int s2 = lo; s2 < hi; s2++) {
        K.site_block[s2] = b;
        const int c0 = site_case_off[s2], c1 = site_case_off[s2 + 1];
        double wsum = 0.0;
        for (int c = c0; c < c1; c++) wsum += case_pauli_off[c + 1] - case_pauli_off[c];
        mu += 32.0 * std::min(1.0, site_prob[s2]) * (c1 > c0 ? wsum / (c1 - c0) : 0.0);
      }
      const int cap = (int)std::ceil(mu + 8.0 * std::sqrt(mu) + 16.0);
      K.block_hi.push_back(hi);
      K.block_cap.push_back(cap);
      K.row_off.push_back(K.rows);
      K.rows += cap;
      K.capmax = std::max(K.capmax, cap);
      b++;
      K.nblocks = b;
    }
  K.pslot.assign(paulis.size() + 1, 0);
  std::vector<int> phys(2 * n);
  for (int v = 0; v < 2 * n; v++) phys[v] = v;
  auto X = [&](int q) { return phys[q]; };
  auto Z = [&](int q) { return phys[n + q]; };
  std::ostringstream o;
  auto f = [&](int slot) {
    std::ostringstream t;
    t << "F[" << slot * 32 << "]";
    return t.str();
  };
  const int R = d.record_count;
  o << "#include \"fs_jit_kernels.cuh\"\n";
  const char* mb = getenv("FS_JIT_MINBLOCKS");
  o << "extern \"C\" __global__ void __launch_bounds__(128, " << (mb ? atoi(mb) : 3) << ") fs_jit_frame(fs::DevProg P, fs::RunArgs A, "
       "const uint16_t* __restrict__ pslot, const uint32_t* __restrict__ fent, const uint32_t* __restrict__ bcount, "
       "const uint32_t* __restrict__ ntot) {\n";
  o << "  extern __shared__ uint32_t smem[];\n";
  o << "  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;\n";
  o << "  uint32_t* F = smem + wib * " << (K.nslots + K.stage) * 32 << " + lane;\n";
  o << "  uint32_t* stage = smem + wib * " << (K.nslots + K.stage) * 32 << " + " << K.nslots * 32 << ";\n";
  o << "  const uint64_t word0 = A.shot0 >> 5;\n";
  o << "  const uint64_t seed = A.seed;\n";
  o << "  for (uint32_t w = (blockIdx.x * 4 + wib) * 32 + lane; w < A.W; w += gridDim.x * 4 * 32) {\n";
  o << "    const uint64_t wabs = word0 + w;\n";
  o << "    const uint64_t nleft = A.nshots - (uint64_t)w * 32;\n";
  o << "    const uint32_t valid = nleft >= 32 ? 0xFFFFFFFFu : ((1u << nleft) - 1u);\n";
  o << "    uint32_t alive = valid;\n";
  o << "#pragma unroll\n    for (int s = 0; s < " << K.nslots << "; s++) F[s * 32] = 0u;\n";
  for (int s = 0; s < d.num_slots; s++) o << "    uint32_t r" << s << " = 0u;\n";
  for (int j = 0; j < d.num_observables; j++) o << "    uint32_t ob" << j << " = 0u;\n";
  o << "    uint4 cb = make_uint4(0u, 0u, 0u, 0u);\n";
  // faults come from the pre-generated per-word list (noise_list_kernel); an overflowed list
  // (count == ~0) falls back to generating the word's stream in place
  // stage the word's fault entries into shared memory with full-row loads (all lanes read
  // entry row t together), and prefetch the per-block counts
  o << "    const uint32_t nt_ = ntot[w];\n    const bool fover = nt_ == 0xFFFFFFFFu;\n";
  o << "    fs::FaultBuffer<fs::kFaultCap> fbuf;\n    if (fover) fbuf.init(P, seed, wabs);\n";
  o << "    uint32_t fcur = 0;\n";
  o << "    {\n      const uint32_t mine = fover ? 0u : min(nt_, " << K.stage << "u);\n";
  o << "      uint32_t tmax = mine;\n";
  o << "      for (int o_ = 16; o_; o_ >>= 1) tmax = max(tmax, __shfl_xor_sync(__activemask(), tmax, o_));\n";
  o << "      for (uint32_t t = 0; t < tmax; t++) if (t < mine) stage[t * 32 + lane] = __ldg(fent + (size_t)t * A.ostride + w);\n";
  o << "    }\n";
  for (int b = 0; b < K.nblocks; b++) o << "    const uint32_t nbk" << b << " = fover ? 0u : __ldg(bcount + (size_t)" << b << " * A.ostride + w);\n";
  auto put_record = [&](int rec, const std::string& expr) {
    const int col = record_out[rec], sl = bit_slot[rec];
    o << "    { const uint32_t rw = " << expr << ";";
    if (col >= 0) o << " A.meas[(size_t)" << col << " * A.ostride + w] = rw & alive;";
    if (sl >= 0) o << " r" << sl << " = rw;";
    o << " }\n";
  };
  int coin_blk = -1;
  int nblk = 0;  // NoiseBlock ordinal
  for (int i = 0; i < d.num_instrs; i++) {
    const int* I = ins_all.data() + (size_t)i * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]);
    const bool flip = FS_FLIP(I[0]);
    switch (op) {
      case FS_OP_FRAME:
        for (int j = 0; j < I[2]; j++) {
          const uint32_t g = gates[I[1] + j];
          const int a = FS_GATE_A(g), b = FS_GATE_B(g);
          switch (FS_GATE_G(g)) {
            case FS_G_H: std::swap(phys[a], phys[n + a]); break;
            case FS_G_S:
            case FS_G_SDAG: o << "    " << f(Z(a)) << " ^= " << f(X(a)) << ";\n"; break;
            case FS_G_CX:
              o << "    " << f(X(b)) << " ^= " << f(X(a)) << "; " << f(Z(a)) << " ^= " << f(Z(b)) << ";\n";
              break;
            case FS_G_CZ:
              o << "    " << f(Z(b)) << " ^= " << f(X(a)) << "; " << f(Z(a)) << " ^= " << f(X(b)) << ";\n";
              break;
            case FS_G_SWAP:
              std::swap(phys[a], phys[b]);
              std::swap(phys[n + a], phys[n + b]);
              break;
          }
        }
        break;
      case FS_OP_MEAS_DSTATIC:
        put_record(I[3], f(X(I[1])) + (flip ? " ^ 0xFFFFFFFFu" : ""));
        break;
      case FS_OP_MEAS_DRANDOM: {
        const int virt = I[1], ord = I[2];
        if (ord / 4 != coin_blk) {
          coin_blk = ord / 4;
          o << "    cb = fs::coin_block(seed, wabs, " << coin_blk << ");\n";
        }
        const char* comp[4] = {"cb.x", "cb.y", "cb.z", "cb.w"};
        o << "    { const uint32_t coin = " << comp[ord & 3] << "; const uint32_t pw = " << f(Z(virt)) << ";";
        o << " " << f(Z(virt)) << " = pw ^ coin;";
        const int col = record_out[I[3]], sl = bit_slot[I[3]];
        o << " const uint32_t rw = coin ^ pw" << (flip ? " ^ 0xFFFFFFFFu" : "") << ";";
        if (col >= 0) o << " A.meas[(size_t)" << col << " * A.ostride + w] = rw & alive;";
        if (sl >= 0) o << " r" << sl << " = rw;";
        o << " }\n";
        // fx_new = fz_old ^ coin (already in the old z slot), fz_new = fx_old: rename
        std::swap(phys[virt], phys[n + virt]);
        break;
      }
      case FS_OP_COND_FRAME: {
        const int sl = bit_slot[I[3]];
        for (int j = I[1]; j < I[1] + I[2]; j++) {
          const uint32_t e = paulis[j];
          const int q = FS_PAULI_Q(e);
          o << "    " << f(FS_PAULI_Z(e) ? Z(q) : X(q)) << " ^= r" << sl << ";\n";
        }
        break;
      }
      case FS_OP_NOISE: {
        for (int s = I[1]; s < I[2]; s++)
          for (int c = site_case_off[s]; c < site_case_off[s + 1]; c++)
            for (int j = case_pauli_off[c]; j < case_pauli_off[c + 1]; j++) {
              const uint32_t e = paulis[j];
              const int q = FS_PAULI_Q(e);
              K.pslot[j] = (uint16_t)(FS_PAULI_Z(e) ? Z(q) : X(q));
            }
        o << "    if (!fover) fs::jit_apply_faults(F, stage, pslot, lane, fcur, nbk" << nblk
          << "); else fs::jit_noise_block(P, F, pslot, fbuf, " << I[2] << ");\n";
        nblk++;
        break;
      }
      case FS_OP_DETECTOR:
      case FS_OP_OBSERVABLE: {
        std::ostringstream e;
        e << "0u";
        for (int j = 0; j < I[3]; j++) e << " ^ r" << bit_slot[reclists[I[2] + j]];
        if (op == FS_OP_DETECTOR) {
          const int sl = bit_slot[R + I[1]];
          o << "    { const uint32_t dw = " << e.str() << "; A.det[(size_t)" << I[1] << " * A.ostride + w] = dw & alive;";
          if (sl >= 0) o << " r" << sl << " = dw;";
          o << " }\n";
        } else {
          o << "    ob" << I[1] << " ^= (" << e.str() << ") & alive;\n";
        }
        break;
      }
      case FS_OP_POSTSELECT: {
        const int bid = I[1] == 0 ? R + I[2] : I[2];
        o << "    alive &= ~((r" << bit_slot[bid] << (I[3] ? " ^ 0xFFFFFFFFu" : "") << ") & alive);\n";
        break;
      }
      default:
        break;  // GammaRot: global phase only
    }
  }
  for (int j = 0; j < d.num_observables; j++)
    o << "    A.obs[(size_t)" << j << " * A.ostride + w] = ob" << j << " & valid;\n";
  o << "    A.accepted[w] = alive & valid;\n    A.error[w] = 0u;\n  }\n}\n";
  K.src = o.str();
  return K;
}


// ------------------------------------------------------------------------------------------
// Program-specialised kernel for the general engine (0 < k_max <= 7, no PostSelect, Philox,
// free sampling): warp = 32-shot word, lane = shot.  Frame words are per-lane registers holding
// the same (warp-uniform) value in every lane, with H / SWAP / MeasDormantRandom's x<->z as
// compile-time renaming; noise faults are applied through a per-warp shared-memory shadow of the
// touched slots.  The active array is in registers (k_max <= 4) or in shared memory at constant
// offsets (interleaved [i][lane]); every array operation is unrolled with constant indices and
// uses the same rounding sequence as the interpreter (bit-identical results).
inline std::string hexd(double v) {
  char b[64];
  if (v != v || v - v != 0.0) {  // NaN / inf: spelled by their bits (NVRTC has no literal for them)
    unsigned long long u;
    memcpy(&u, &v, sizeof u);
    snprintf(b, sizeof b, "__longlong_as_double(0x%016llxULL)", u);
  } else {
    snprintf(b, sizeof b, "%a", v);
  }
  return b;
}

struct GeneralKernelSource {
  std::string src;
  std::vector<uint16_t> pslot;
  int nslots = 0, cap_log2 = 0, nblocks = 0;
  bool arr_regs = true;
  int nreg = 0;  // smem arrays: amplitudes [0, nreg) live in registers, the rest in shared memory
  std::vector<int32_t> site_block;
};

inline GeneralKernelSource gen_general_kernel(const fs_prog_desc& d, const std::vector<int32_t>& ins_all,
                                              const std::vector<uint32_t>& gates, const std::vector<uint32_t>& paulis,
                                              const std::vector<int32_t>& reclists,
                                              const std::vector<int32_t>& record_out,
                                              const std::vector<int32_t>& bit_slot,
                                              const std::vector<int32_t>& case_pauli_off,
                                              const std::vector<int32_t>& site_case_off,
                                              const std::vector<double>& fparams) {
  GeneralKernelSource K;
  const int n = d.n, R = d.record_count;
  K.nslots = 2 * n;
  K.cap_log2 = d.k_max;
  K.arr_regs = d.k_max <= 4;
  if (const char* e = getenv("FS_GJIT_SMEM")) K.arr_regs = K.arr_regs && atoi(e) == 0;  // tuning
  // larger arrays: the low half (at most 32) of the amplitudes stays in registers, the rest in shared
  // memory (config 0, k = 6: 0.053 -> 0.040 ms per 1e5 shots; 16 or 48 registers-resident: 0.042 / 0.041)
  // (with the noiseless prefix executed per shot, config 0 at k = 6: 32 register-resident -> 0.077
  // ms per 1e5 shots (spills), 24 -> 0.057, 16 -> 0.059, 8 -> 0.070)
  K.nreg = K.arr_regs ? (1 << d.k_max) : std::min(24, (1 << d.k_max) / 2);
  if (const char* e = getenv("FS_GJIT_NREG")) if (!K.arr_regs) K.nreg = std::max(0, std::min(atoi(e), (1 << d.k_max) - 1));
  K.pslot.assign(paulis.size() + 1, 0);
  K.site_block.assign(d.num_sites + 1, 0);
  for (int i = 0, b = 0; i < d.num_instrs; i++)
    if (FS_OPCODE(ins_all[(size_t)i * FS_INS_WORDS]) == FS_OP_NOISE) {
      for (int s2 = ins_all[(size_t)i * FS_INS_WORDS + 1]; s2 < ins_all[(size_t)i * FS_INS_WORDS + 2]; s2++) K.site_block[s2] = b;
      K.nblocks = ++b;
    }
  std::vector<int> phys(2 * n);
  for (int v = 0; v < 2 * n; v++) phys[v] = v;
  auto X = [&](int q) { return phys[q]; };
  auto Z = [&](int q) { return phys[n + q]; };
  auto f = [&](int slot) { return "f" + std::to_string(slot); };
  auto A = [&](int i) {
    return i < K.nreg ? "a" + std::to_string(i) : "AR[" + std::to_string((i - K.nreg) * 32) + "]";
  };
  auto C = [&](int off) { return "make_double2(" + hexd(fparams[off]) + ", " + hexd(fparams[off + 1]) + ")"; };
  const int cap = 1 << d.k_max;
  std::ostringstream o;
  o << "#include \"fs_jit_kernels.cuh\"\n";
  o << "#define cmul fs::cmul_f\nusing fs::cadd; using fs::csub; using fs::cscale; using fs::cnorm2;\n";
  const char* gmb = getenv("FS_GJIT_MB");
  // register arrays: 4 blocks of 4 warps per SM (config 2: 2.38 -> 2.30 ms; 3 blocks leave 168
  // registers, 5 and more spill)
  o << "extern \"C\" __global__ void __launch_bounds__(" << (K.arr_regs ? 128 : 64) << ", " << (gmb ? atoi(gmb) : (K.arr_regs ? 4 : 1))
    << ") fs_jit_general(fs::DevProg P, fs::RunArgs A, const uint16_t* __restrict__ pslot, "
       "const uint32_t* __restrict__ fent, const uint32_t* __restrict__ bcount, const uint32_t* __restrict__ ntot) {\n";
  o << "  extern __shared__ __align__(16) unsigned char smem[];\n";
  o << "  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;\n";
  const int fs_words = (2 * n + 3) / 4 * 4;
  o << "  uint32_t* Fs = reinterpret_cast<uint32_t*>(smem) + wib * " << fs_words << ";\n";
  if (!K.arr_regs)
    o << "  double2* AR = reinterpret_cast<double2*>(smem + nw * " << fs_words * 4 << ") + wib * " << (cap - K.nreg) * 32
      << " + lane;\n";
  o << "  const uint64_t word0 = A.shot0 >> 5;\n  const uint64_t seed = A.seed;\n";
  o << "  for (uint32_t w = blockIdx.x * nw + wib; w < A.W; w += gridDim.x * nw) {\n";
  o << "    const uint64_t si = (uint64_t)w * 32 + lane;\n    const bool valid = si < A.nshots;\n";
  o << "    const uint64_t shot = A.shot0 + si;\n    const uint64_t wabs = word0 + w;\n";
  o << "    const uint32_t validm = __ballot_sync(0xFFFFFFFFu, valid);\n";
  o << "    uint32_t alive = validm, errm = 0;\n";
  for (int sl = 0; sl < 2 * n; sl++) o << "    uint32_t " << f(sl) << " = 0u;\n";
  for (int sl = 0; sl < d.num_slots; sl++) o << "    uint32_t r" << sl << " = 0u;\n";
  for (int j = 0; j < d.num_observables; j++) o << "    uint32_t ob" << j << " = 0u;\n";
  // the initial amplitude 1 is opaque to the compiler (asm): the array work of a noiseless
  // prefix (config 0: the six Expands before the first random draw) is executed per shot, never
  // constant-folded into the kernel
  o << "    double one_;\n    asm volatile(\"mov.b64 %0, 0x3FF0000000000000;\" : \"=d\"(one_));\n";
  for (int i = 0; i < K.nreg; i++) o << "    double2 a" << i << " = make_double2(" << (i == 0 ? "one_" : "0.0") << ", 0.0);\n";
  if (K.nreg == 0) o << "    AR[0] = make_double2(one_, 0.0);\n";
  o << "    uint4 cb = make_uint4(0u, 0u, 0u, 0u);\n";
  // no NoiseBlock: no fault lists (the launcher skips their kernel)
  if (K.nblocks) o << "    const uint32_t nt_ = ntot[w];\n    const bool fover = nt_ == 0xFFFFFFFFu;\n    uint32_t fcur = 0;\n";
  else o << "    const bool fover = false;\n    uint32_t fcur = 0;\n";
  o << "    fs::WordFaultGen gen;\n    int psite = -1, plane = 0, pcase = 0;\n    if (fover) gen.init(seed, wabs);\n";
  auto put_record = [&](int rec, const std::string& expr) {
    const int col = record_out[rec], sl = bit_slot[rec];
    o << "    { const uint32_t rw = " << expr << ";";
    if (col >= 0) o << " if (lane == 0) A.meas[(size_t)" << col << " * A.ostride + w] = rw & alive;";
    if (sl >= 0) o << " r" << sl << " = rw;";
    o << " }\n";
  };
  int coin_blk = -1, nblk = 0;
  for (int i = 0; i < d.num_instrs; i++) {
    const int* I = ins_all.data() + (size_t)i * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]);
    const bool flip = FS_FLIP(I[0]);
    const std::string flipm = flip ? " ^ 0xFFFFFFFFu" : "";
    switch (op) {
      case FS_OP_FRAME:
        for (int j = 0; j < I[2]; j++) {
          const uint32_t g = gates[I[1] + j];
          const int a = FS_GATE_A(g), b = FS_GATE_B(g);
          switch (FS_GATE_G(g)) {
            case FS_G_H: std::swap(phys[a], phys[n + a]); break;
            case FS_G_S: case FS_G_SDAG: o << "    " << f(Z(a)) << " ^= " << f(X(a)) << ";\n"; break;
            case FS_G_CX: o << "    " << f(X(b)) << " ^= " << f(X(a)) << "; " << f(Z(a)) << " ^= " << f(Z(b)) << ";\n"; break;
            case FS_G_CZ: o << "    " << f(Z(b)) << " ^= " << f(X(a)) << "; " << f(Z(a)) << " ^= " << f(X(b)) << ";\n"; break;
            case FS_G_SWAP: std::swap(phys[a], phys[b]); std::swap(phys[n + a], phys[n + b]); break;
          }
        }
        break;
      case FS_OP_ARRAY_GATE: {
        const int g = I[1], va = I[2], vb = I[3], a = I[4], b = I[5], size = 1 << I[6];
        if (g == FS_G_S || g == FS_G_SDAG) {
          for (int j = 0; j < size; j++)
            if ((j >> a) & 1) {  // x (+/-)i: a swap and a sign flip
              if (g == FS_G_S) o << "    " << A(j) << " = make_double2(-" << A(j) << ".y, " << A(j) << ".x);\n";
              else o << "    " << A(j) << " = make_double2(" << A(j) << ".y, -" << A(j) << ".x);\n";
            }
          o << "    " << f(Z(va)) << " ^= " << f(X(va)) << ";\n";
        } else if (g == FS_G_H) {
          const int st = 1 << a;
          for (int j = 0; j < size; j++)
            if (!((j >> a) & 1))
              o << "    { const double2 lo = " << A(j) << ", hi = " << A(j + st) << "; " << A(j)
                << " = cscale(cadd(lo, hi), fs::kInvSqrt2); " << A(j + st) << " = cscale(csub(lo, hi), fs::kInvSqrt2); }\n";
          std::swap(phys[va], phys[n + va]);
        } else if (g == FS_G_CX) {
          for (int j = 0; j < size; j++)
            if (((j >> a) & 1) && !((j >> b) & 1))
              o << "    { const double2 t0 = " << A(j) << "; " << A(j) << " = " << A(j | (1 << b)) << "; " << A(j | (1 << b)) << " = t0; }\n";
          o << "    " << f(X(vb)) << " ^= " << f(X(va)) << "; " << f(Z(va)) << " ^= " << f(Z(vb)) << ";\n";
        } else if (g == FS_G_CZ) {
          for (int j = 0; j < size; j++)
            if (((j >> a) & 1) && ((j >> b) & 1)) o << "    " << A(j) << " = make_double2(-" << A(j) << ".x, -" << A(j) << ".y);\n";
          o << "    " << f(Z(vb)) << " ^= " << f(X(va)) << "; " << f(Z(va)) << " ^= " << f(X(vb)) << ";\n";
        }
        break;
      }
      case FS_OP_EXPAND: {
        const int size = 1 << I[6];
        o << "    { const int par = (" << f(X(I[1])) << " >> lane) & 1;\n";
        o << "      const double2 ph0 = par ? " << C(I[5] + 4) << " : " << C(I[5]) << ";\n";
        o << "      const double2 ph1 = par ? " << C(I[5] + 6) << " : " << C(I[5] + 2) << ";\n";
        for (int j = 0; j < size; j++)
          o << "      { const double2 v = " << A(j) << "; " << A(j) << " = cmul(v, ph0); " << A(size + j) << " = cmul(v, ph1); }\n";
        o << "    }\n";
        break;
      }
      case FS_OP_ARRAY_ROT: {
        const int a = I[2], size = 1 << I[6];
        o << "    { const int par = (" << f(X(I[1])) << " >> lane) & 1;\n";
        o << "      const double2 ph0 = par ? " << C(I[5] + 2) << " : " << C(I[5]) << ";\n";
        o << "      const double2 ph1 = par ? " << C(I[5]) << " : " << C(I[5] + 2) << ";\n";
        for (int j = 0; j < size; j++) o << "      " << A(j) << " = cmul(" << A(j) << ", " << (((j >> a) & 1) ? "ph1" : "ph0") << ");\n";
        o << "    }\n";
        break;
      }
      case FS_OP_GAMMA_ROT:
        break;  // global phase: no effect on records
      case FS_OP_MEAS_DSTATIC:
        put_record(I[3], f(X(I[1])) + flipm);
        break;
      case FS_OP_MEAS_DRANDOM: {
        const int virt = I[1], ord = I[2];
        if (ord / 4 != coin_blk) {
          coin_blk = ord / 4;
          o << "    cb = fs::coin_block(seed, wabs, " << coin_blk << ");\n";
        }
        const char* comp[4] = {"cb.x", "cb.y", "cb.z", "cb.w"};
        o << "    { const uint32_t coin = " << comp[ord & 3] << "; const uint32_t pw = " << f(Z(virt)) << "; "
          << f(Z(virt)) << " = pw ^ coin;";
        const int col = record_out[I[3]], sl = bit_slot[I[3]];
        o << " const uint32_t rw = coin ^ pw" << flipm << ";";
        if (col >= 0) o << " if (lane == 0) A.meas[(size_t)" << col << " * A.ostride + w] = rw & alive;";
        if (sl >= 0) o << " r" << sl << " = rw;";
        o << " }\n";
        std::swap(phys[virt], phys[n + virt]);
        break;
      }
      case FS_OP_MEAS_COLLAPSE: {
        const int virt = I[1], a = I[2], rec = I[3], size = 1 << I[6], half = size >> 1, st = 1 << a;
        const int po = I[4] >> 8, pc = I[4] & 0xFF;
        for (int j = 0; j < pc; j++) {
          const uint32_t g = gates[po + j];
          const int q = FS_GATE_A(g);
          if (FS_GATE_G(g) == FS_G_H) std::swap(phys[q], phys[n + q]);
          else o << "    " << f(Z(q)) << " ^= " << f(X(q)) << ";\n";
        }
        const int fo = I[5];
        // complex products with a compile-time-real (or imaginary) factor: the zero component's
        // products vanish from cmul_f exactly, so two multiplies give the same doubles
        auto cm = [&](int uoff, const std::string& u, const std::string& a) -> std::string {
          if (fparams[uoff + 1] == 0.0) return "fs::cmul_re(" + u + ".x, " + a + ")";
          if (fparams[uoff] == 0.0) return "fs::cmul_im(" + u + ".y, " + a + ")";
          return "cmul(" + u + ", " + a + ")";
        };
        const bool k0re = fparams[fo + 1] == 0.0 && fparams[fo + 5] == 0.0;
        const bool k1re = fparams[fo + 3] == 0.0 && fparams[fo + 7] == 0.0;
        o << "    {\n      const double2 u00 = " << C(fo) << ", u01 = " << C(fo + 2) << ", u10 = " << C(fo + 4)
          << ", u11 = " << C(fo + 6) << ";\n";
        o << "      const int parity = (" << f(X(virt)) << " >> lane) & 1;\n";
        o << "      double p1 = 0.0, p_all = 0.0;\n";
        if (size == 2) {
          o << "      { const double2 b0 = cadd(" << cm(fo, "u00", A(0)) << ", " << cm(fo + 2, "u01", A(1)) << "); const double2 b1 = cadd("
            << cm(fo + 4, "u10", A(0)) << ", " << cm(fo + 6, "u11", A(1)) << "); p1 = cnorm2(b1); p_all = __dadd_rn(p1, cnorm2(b0)); }\n";
        } else if (size <= 16) {
          for (int j = 0; j < size; j++)
            if (!((j >> a) & 1))
              o << "      { const double2 a0_ = " << A(j) << ", a1_ = " << A(j + st)
                << "; const double q1 = cnorm2(cadd(" << cm(fo + 4, "u10", "a0_") << ", " << cm(fo + 6, "u11", "a1_")
                << ")); const double2 b0 = cadd(" << cm(fo, "u00", "a0_") << ", " << cm(fo + 2, "u01", "a1_") << "); "
                   "p1 = __dadd_rn(p1, q1); p_all = __dadd_rn(p_all, __dadd_rn(q1, cnorm2(b0))); }\n";
        } else {
          for (int j = 0; j < size; j++)
            if (!((j >> a) & 1))
              o << "      p1 = __dadd_rn(p1, cnorm2(cadd(cmul(" << A(j) << ", u10), cmul(u11, " << A(j + st) << "))));\n";
          for (int j = 0; j < size; j++) o << "      p_all = __dadd_rn(p_all, cnorm2(" << A(j) << "));\n";
        }
        o << "      const bool bad = p1 != p1;\n";
        o << "      p1 = p_all > 0 ? __ddiv_rn(p1, p_all) : 0.0;\n      if (p1 < 0.0) p1 = 0.0; else if (p1 > 1.0) p1 = 1.0;\n";
        o << "      const uint4 bo = fs::philox((uint32_t)shot, (uint32_t)(shot >> 32), " << i << "u, fs::TAG_BORN << 24, seed);\n";
        o << "      int br = fs::u64_to_unit(((uint64_t)bo.y << 32) | bo.x) < p1 ? 1 : 0;\n";
        o << "      double pb = br ? p1 : __dsub_rn(1.0, p1);\n";
        o << "      if (pb < fs::kBranchFloor) { br ^= 1; pb = __dsub_rn(1.0, pb); }\n";
        o << "      const double scale = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(pb, p_all)));\n";
        o << "      const double2 k0 = br == 0 ? cscale(u00, scale) : cscale(u10, scale);\n";
        o << "      const double2 k1 = br == 0 ? cscale(u01, scale) : cscale(u11, scale);\n";
        for (int j = 0; j < half; j++) {
          const int i0 = ((j >> a) << (a + 1)) | (j & (st - 1));
          o << "      " << A(j) << " = cadd(" << (k0re ? "fs::cmul_re(k0.x, " + A(i0) + ")" : "cmul(k0, " + A(i0) + ")") << ", "
            << (k1re ? "fs::cmul_re(k1.x, " + A(i0 + st) + ")" : "cmul(k1, " + A(i0 + st) + ")") << ");\n";
        }
        o << "      const uint32_t badw = __ballot_sync(0xFFFFFFFFu, bad && ((alive >> lane) & 1));\n";
        o << "      errm |= badw; alive &= ~badw;\n";
        o << "      const uint32_t recw = __ballot_sync(0xFFFFFFFFu, (br ^ parity ^ " << (flip ? 1 : 0) << ") != 0);\n";
        o << "      const uint32_t brw = __ballot_sync(0xFFFFFFFFu, br != 0);\n";
        o << "      " << f(X(virt)) << " ^= brw;\n";
        const int col = record_out[rec], sl = bit_slot[rec];
        if (col >= 0) o << "      if (lane == 0) A.meas[(size_t)" << col << " * A.ostride + w] = recw & alive;\n";
        if (sl >= 0) o << "      r" << sl << " = recw;\n";
        o << "    }\n";
        break;
      }
      case FS_OP_COND_FRAME: {
        const int sl = bit_slot[I[3]];
        for (int j = I[1]; j < I[1] + I[2]; j++) {
          const uint32_t e = paulis[j];
          const int q = FS_PAULI_Q(e);
          o << "    " << f(FS_PAULI_Z(e) ? Z(q) : X(q)) << " ^= r" << sl << ";\n";
        }
        break;
      }
      case FS_OP_NOISE: {
        // touched physical slots of this block; pslot under the current renaming
        std::vector<int> touched;
        for (int s2 = I[1]; s2 < I[2]; s2++)
          for (int c = site_case_off[s2]; c < site_case_off[s2 + 1]; c++)
            for (int j = case_pauli_off[c]; j < case_pauli_off[c + 1]; j++) {
              const uint32_t e = paulis[j];
              const int q = FS_PAULI_Q(e);
              const int sl = FS_PAULI_Z(e) ? Z(q) : X(q);
              K.pslot[j] = (uint16_t)sl;
              touched.push_back(sl);
            }
        std::sort(touched.begin(), touched.end());
        touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
        o << "    {\n";
        for (int sl : touched) o << "      Fs[" << sl << "] = " << f(sl) << ";\n";
        o << "      __syncwarp();\n      if (lane == 0) {\n";
        o << "        if (!fover) {\n          const uint32_t nb_ = __ldg(bcount + (size_t)" << nblk << " * A.ostride + w);\n";
        o << "          for (uint32_t t = 0; t < nb_; t++) {\n";
        o << "            const uint32_t e = __ldg(fent + (size_t)(fcur + t) * A.ostride + w);\n";
        o << "            const uint32_t bit = 1u << (e & 31);\n            const int off = (int)(e >> 10), cnt = (int)((e >> 5) & 31);\n";
        o << "            for (int j = 0; j < cnt; j++) Fs[__ldg(pslot + off + j)] ^= bit;\n          }\n";
        o << "          fcur += nb_;\n        } else {\n";
        o << "          fs::gjit_noise_fallback(P, Fs, pslot, gen, psite, plane, pcase, " << I[2] << ");\n";
        o << "        }\n      }\n      __syncwarp();\n";
        for (int sl : touched) o << "      " << f(sl) << " = Fs[" << sl << "];\n";
        o << "      __syncwarp();\n";
        o << "    }\n";
        nblk++;
        break;
      }
      case FS_OP_DETECTOR:
      case FS_OP_OBSERVABLE: {
        std::ostringstream e;
        e << "0u";
        for (int j = 0; j < I[3]; j++) e << " ^ r" << bit_slot[reclists[I[2] + j]];
        if (op == FS_OP_DETECTOR) {
          const int sl = bit_slot[R + I[1]];
          o << "    { const uint32_t dw = " << e.str() << "; if (lane == 0) A.det[(size_t)" << I[1] << " * A.ostride + w] = dw & alive;";
          if (sl >= 0) o << " r" << sl << " = dw;";
          o << " }\n";
        } else {
          o << "    ob" << I[1] << " ^= (" << e.str() << ") & alive;\n";
        }
        break;
      }
      default:
        break;
    }
  }
  o << "    if (lane == 0) {\n";
  for (int j = 0; j < d.num_observables; j++) o << "      A.obs[(size_t)" << j << " * A.ostride + w] = ob" << j << " & validm;\n";
  o << "      A.accepted[w] = alive & validm;\n      A.error[w] = errm;\n      if (errm) atomicMax(A.status, FS_ERR_SHOT_NAN);\n    }\n";
  o << "    __syncwarp();\n  }\n}\n";
  K.src = o.str();
  return K;
}

struct Compiled {
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  double compile_s = 0.0;
  size_t cubin_bytes = 0;
  std::string log;
};

inline std::string compile(const std::string& src, const std::string& incdir, Compiled& out,
                           const char* kname = "fs_jit_frame") {
  Api& A = api();
  if (!A.ok) return "JIT unavailable: " + A.why;
  if (const char* dump = getenv("FS_JIT_DUMP")) {  // debugging: keep the generated source
    if (FILE* f = fopen((std::string(dump) + "/" + kname + ".cu").c_str(), "w")) {
      fwrite(src.data(), 1, src.size(), f);
      fclose(f);
    }
  }
  void* prog = nullptr;
  if (A.nvrtcCreateProgram(&prog, src.c_str(), (std::string(kname) + ".cu").c_str(), 0, nullptr, nullptr) != 0)
    return "nvrtcCreateProgram failed";
  std::string inc = "-I" + incdir;
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", inc.c_str(), "-DFS_JIT=1"};
  int rc = A.nvrtcCompileProgram(prog, 5, opts);
  size_t lsz = 0;
  A.nvrtcGetProgramLogSize(prog, &lsz);
  std::string log(lsz, '\0');
  if (lsz) A.nvrtcGetProgramLog(prog, &log[0]);
  out.log = log;
  if (rc != 0) {
    A.nvrtcDestroyProgram(&prog);
    return "NVRTC compile failed: " + log.substr(0, 2000);
  }
  size_t csz = 0;
  A.nvrtcGetCUBINSize(prog, &csz);
  std::vector<char> cubin(csz);
  A.nvrtcGetCUBIN(prog, cubin.data());
  A.nvrtcDestroyProgram(&prog);
  out.cubin_bytes = csz;
  CUresult r = A.cuModuleLoadData(&out.mod, cubin.data());
  if (r != 0) return "cuModuleLoadData failed (" + std::to_string(r) + ")";
  r = A.cuModuleGetFunction(&out.fn, out.mod, kname);
  if (r != 0) return "cuModuleGetFunction failed (" + std::to_string(r) + ")";
  return "";
}

}  // namespace fsjit
