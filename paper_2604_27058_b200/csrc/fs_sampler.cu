// fs_sampler.cu -- C ABI (include/fs_sampler.h) over the sm_100a engines.
//
//   engine 1 (fs_frame.cuh)   frame-only programs: lane = 32-shot word, 1024 shots per warp
//   engine 0 (fs_general.cuh) everything else: warp = 32-shot word, lane = shot
//
// No CPU fallback exists: if CUDA is unavailable every entry point fails with FS_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fs_frame.cuh"
#include "fs_general.cuh"

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

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct fs_prog {
  fs_prog_desc desc;  // scalar fields only (pointers refer to host memory of the creator)
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
  // pointers of the creator's arrays are not retained
  p->desc.instrs = nullptr;
  *out = p;
  return FS_OK;
}

extern "C" void fs_program_destroy(fs_prog* p) {
  if (!p) return;
  cudaFree(p->dbuf);
  cudaFree(p->scratch);
  cudaFree(p->d_status);
  cudaFree(p->stage);
  cudaFree(p->d_counts);
  delete p;
}

static bool wants_general(const fs_prog* p, uint32_t flags, const fs_trace_out* tout) {
  if (p->dp.k_max > 0) return true;
  if (flags & (FS_RNG_SPLITMIX | FS_FORCE_GENERAL)) return true;
  if (tout && (tout->gamma || tout->amps || tout->draws)) return true;
  return false;
}

extern "C" int fs_program_engine(const fs_prog* p, uint32_t flags) {
  if (!p) return set_error(FS_ERR_ARG, "null program");
  return wants_general(p, flags, nullptr) ? 0 : 1;
}

namespace {

template <class K>
int occupancy_blocks(K kernel, int threads, size_t smem) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess) return 1;
  return std::max(nb, 1);
}

int launch(fs_prog* p, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags, const fs_trace_in* tin,
           const fs_sample_out* out, const fs_trace_out* tout, cudaStream_t stream) {
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
    if ((a.t_fx == nullptr) != (a.t_fz == nullptr)) return set_error(FS_ERR_ARG, "frame_x/frame_z must both be set");
  }
  a.arr_log2 = dp.k_max;
  if (!out->status) FS_CUDA_TRY(cudaMemsetAsync(p->d_status, 0, sizeof(int), stream));
  const size_t W = a.W;
  a.prezeroed = 0;
  if (dp.has_psel) {  // halted warps may stop early: their remaining output words must read 0
    if (dp.U) FS_CUDA_TRY(cudaMemsetAsync(a.meas, 0, sizeof(uint32_t) * dp.U * W, stream));
    if (dp.D) FS_CUDA_TRY(cudaMemsetAsync(a.det, 0, sizeof(uint32_t) * dp.D * W, stream));
    a.prezeroed = 1;
  }
  const bool general = wants_general(p, flags, tout);
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
    kern<<<(unsigned)grid, threads, smem, stream>>>(dp, a, words_per_warp);
    FS_CUDA_TRY(cudaGetLastError());
    return FS_OK;
  }
  // general engine
  const bool splitmix = flags & FS_RNG_SPLITMIX;
  const int words_per_warp = (int)align_up(2 * dp.n + dp.num_slots + dp.O, 4);
  const size_t words_bytes = (size_t)fs::kGenWarps * words_per_warp * 4;
  const size_t arr_bytes_warp = ((size_t)32 << dp.k_max) * sizeof(double2);
  const bool arr_smem = words_bytes + 16 + fs::kGenWarps * arr_bytes_warp <= kSmemBudget;
  const size_t smem = words_bytes + (arr_smem ? 16 + fs::kGenWarps * arr_bytes_warp : 0);
  if (words_bytes > kSmemBudget) return set_error(FS_ERR_ARG, "program too large for the general engine");
  void (*kern)(fs::DevProg, fs::RunArgs, int);
  if (splitmix) kern = arr_smem ? fs::general_kernel<true, true> : fs::general_kernel<true, false>;
  else kern = arr_smem ? fs::general_kernel<false, true> : fs::general_kernel<false, false>;
  FS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int threads = fs::kGenWarps * 32;
  const size_t blocks_needed = (W + fs::kGenWarps - 1) / fs::kGenWarps;
  const int occ = occupancy_blocks(kern, threads, smem);
  size_t grid = std::min<size_t>(blocks_needed, (size_t)p->num_sms * occ);
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
  kern<<<(unsigned)grid, threads, smem, stream>>>(dp, a, words_per_warp);
  FS_CUDA_TRY(cudaGetLastError());
  return FS_OK;
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
  return launch(p, seed, shot0, nshots, flags, tin, out, tout, static_cast<cudaStream_t>(stream));
}

namespace {
struct Stage {  // device staging carve-out for fs_sample_host
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

extern "C" int fs_sample_host(fs_prog* p, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                              const fs_trace_in* tin, const fs_sample_out* out, const fs_trace_out* tout) {
  if (!p || !out) return set_error(FS_ERR_ARG, "null argument");
  if (nshots == 0) return FS_OK;
  std::lock_guard<std::mutex> lk(p->mu);
  const fs::DevProg& dp = p->dp;
  const size_t W = (nshots + 31) / 32;
  int stop = dp.num_instrs;
  if (tin && tin->stop >= 0 && tin->stop < dp.num_instrs) stop = tin->stop;
  int k_stop = 0;
  if (stop > 0) {
    // schedule lives on the device; the host copy was not retained -> fetch one int
    int ks = 0;
    FS_CUDA_TRY(cudaMemcpy(&ks, dp.schedule + stop - 1, sizeof(int), cudaMemcpyDeviceToHost));
    k_stop = ks;
  }
  const size_t n = (size_t)dp.n;
  // sizes
  size_t need = 0;
  auto acc = [&](size_t b) { need = align_up(need + b, 256); };
  acc(4 * W * dp.U); acc(4 * W * dp.D); acc(4 * W * dp.O); acc(4 * W); acc(4 * W); acc(4);
  const bool has_fm = tin && tin->fault_modes, has_fo = tin && tin->forced;
  if (has_fm) acc(2 * nshots * dp.E);
  if (has_fo) acc(nshots * dp.R);
  if (tout) {
    if (tout->frame_x) { acc(nshots * n); acc(nshots * n); }
    if (tout->gamma) acc(16 * nshots);
    if (tout->amps) acc(16 * nshots * ((size_t)1 << k_stop));
    if (tout->draws) acc(4 * nshots);
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
  }
  FS_CUDA_TRY(cudaStreamSynchronize(s));
  if (out->status) *out->status = status;
  if (status) {
    g_last_error = status == FS_ERR_SHOT_NAN ? "NaN amplitude encountered at an active measurement"
                                             : "forced outcome has probability below BRANCH_FLOOR";
  }
  return status;
}

extern "C" int fs_accumulate(fs_prog* p, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                             int64_t* counts, void* stream_) {
  if (!p || !counts) return set_error(FS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lk(p->mu);
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
    int rc = launch(p, seed, shot0 + s0, ns, flags, nullptr, &o, nullptr, stream);
    if (rc != FS_OK) return rc;
    dim3 grid(std::min<uint32_t>((W + 255) / 256, 64), nrows + 1);
    accumulate_kernel<<<grid, 256, 0, stream>>>(rows, nrows, o.accepted, W, counts);
    FS_CUDA_TRY(cudaGetLastError());
  }
  return FS_OK;
}
