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

#include <cmath>
#include <cstdlib>

#include <sstream>
#include <string>
#include <vector>

namespace fsjit {

constexpr int kJitStage = 64;  // staged fault entries per word (more -> in-place generation)

typedef int CUresult;
typedef void* CUmodule;
typedef void* CUfunction;
typedef void* CUstream;

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

inline Api& api() {
  static Api a;
  static bool init = false;
  if (init) return a;
  init = true;
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
#undef LOAD
  a.ok = true;
  return a;
}

struct FrameKernelSource {
  std::string src;
  std::vector<uint16_t> pslot;  // per Pauli entry: physical slot under the renaming at its block
  int nslots = 0;               // physical frame slots (2n)
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
  o << "  uint32_t* F = smem + wib * " << (K.nslots + kJitStage) * 32 << " + lane;\n";
  o << "  uint32_t* stage = smem + wib * " << (K.nslots + kJitStage) * 32 << " + " << K.nslots * 32 << ";\n";
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
  o << "    {\n      const uint32_t mine = fover ? 0u : min(nt_, " << kJitStage << "u);\n";
  o << "      uint32_t tmax = mine;\n";
  o << "      for (int o_ = 16; o_; o_ >>= 1) tmax = max(tmax, __shfl_xor_sync(__activemask(), tmax, o_));\n";
  o << "      for (uint32_t t = 0; t < tmax; t++) if (t < mine) stage[t * 32 + lane] = __ldg(fent + (size_t)t * A.W + w);\n";
  o << "    }\n";
  for (int b = 0; b < K.nblocks; b++) o << "    const uint32_t nbk" << b << " = fover ? 0u : __ldg(bcount + (size_t)" << b << " * A.W + w);\n";
  auto put_record = [&](int rec, const std::string& expr) {
    const int col = record_out[rec], sl = bit_slot[rec];
    o << "    { const uint32_t rw = " << expr << ";";
    if (col >= 0) o << " A.meas[(size_t)" << col << " * A.W + w] = rw & alive;";
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
        if (col >= 0) o << " A.meas[(size_t)" << col << " * A.W + w] = rw & alive;";
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
          o << "    { const uint32_t dw = " << e.str() << "; A.det[(size_t)" << I[1] << " * A.W + w] = dw & alive;";
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
    o << "    A.obs[(size_t)" << j << " * A.W + w] = ob" << j << " & valid;\n";
  o << "    A.accepted[w] = alive & valid;\n    A.error[w] = 0u;\n  }\n}\n";
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

inline std::string compile(const std::string& src, const std::string& incdir, Compiled& out) {
  Api& A = api();
  if (!A.ok) return "JIT unavailable: " + A.why;
  void* prog = nullptr;
  if (A.nvrtcCreateProgram(&prog, src.c_str(), "fs_jit_frame.cu", 0, nullptr, nullptr) != 0)
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
  r = A.cuModuleGetFunction(&out.fn, out.mod, "fs_jit_frame");
  if (r != 0) return "cuModuleGetFunction failed (" + std::to_string(r) + ")";
  return "";
}

}  // namespace fsjit
