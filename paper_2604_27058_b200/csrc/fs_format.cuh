// fs_format.cuh -- the reference CLI's sample output formats (cli.py:66-69, :94-109) produced on
// the device from shot-bit words, so only the final bytes cross PCIe.
//
// Record bits of a shot = user measurements ++ detectors ++ observables (cli.py:67, :102).  A shot
// is kept when it was accepted or keep_rejected (runtime.py:794-795).  Per kept shot:
//   FS_FMT_01  : '0'/'1' per bit, then " rejected" if keep_rejected and not accepted, then '\n'
//   FS_FMT_BIN : np.packbits(bits, bitorder="little") -> ceil(nbits / 8) bytes
//   FS_FMT_CSV : "<index>,<weight>,<bits>\n"  (index = position in the record stream; the weight
//                text is formatted once on the host, f"{weight:.17g}"; the header is the caller's)
// Three passes: kept flags -> ranks (scan), byte lengths -> offsets (scan), write.
#pragma once
#include <cstdint>

namespace fs {

struct FmtArgs {
  const uint32_t* meas;  // [U][W]
  const uint32_t* det;   // [D][W]
  const uint32_t* obs;   // [O][W]
  const uint32_t* accepted;
  uint64_t n;
  uint32_t W;
  int U, D, O;
  int format;  // FS_FMT_*
  int keep_rejected;
  uint64_t index0;
  const char* weight;  // device copy of the weight text
  int wlen;
};

__device__ __forceinline__ uint32_t fmt_bit(const FmtArgs& F, int r, uint64_t s) {
  const uint32_t* row;
  if (r < F.U) row = F.meas + (size_t)r * F.W;
  else if (r < F.U + F.D) row = F.det + (size_t)(r - F.U) * F.W;
  else row = F.obs + (size_t)(r - F.U - F.D) * F.W;
  return (row[s >> 5] >> (s & 31)) & 1u;
}

__device__ __forceinline__ bool fmt_accepted(const FmtArgs& F, uint64_t s) {
  return (F.accepted[s >> 5] >> (s & 31)) & 1u;
}

__device__ __forceinline__ int dec_digits(uint64_t v) {
  int d = 1;
  while (v >= 10) { v /= 10; d++; }
  return d;
}

__global__ void fmt_kept_kernel(FmtArgs F, uint32_t* kept) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= F.n) return;
  kept[s] = (F.keep_rejected || fmt_accepted(F, s)) ? 1u : 0u;
}

__global__ void fmt_len_kernel(FmtArgs F, const uint32_t* kept, const uint32_t* rank, uint64_t* len) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= F.n) return;
  const int nbits = F.U + F.D + F.O;
  uint64_t l = 0;
  if (kept[s]) {
    if (F.format == 0) l = nbits + 1 + ((F.keep_rejected && !fmt_accepted(F, s)) ? 9 : 0);
    else if (F.format == 1) l = (nbits + 7) / 8;
    else l = dec_digits(F.index0 + rank[s]) + 1 + F.wlen + 1 + nbits + 1;
  }
  len[s] = l;
}

__global__ void fmt_write_kernel(FmtArgs F, const uint32_t* kept, const uint32_t* rank, const uint64_t* off,
                                 uint8_t* __restrict__ dst) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= F.n || !kept[s]) return;
  const int nbits = F.U + F.D + F.O;
  uint8_t* o = dst + off[s];
  if (F.format == 1) {  // packbits, little bit order
    uint32_t byte = 0;
    for (int r = 0; r < nbits; r++) {
      byte |= fmt_bit(F, r, s) << (r & 7);
      if ((r & 7) == 7 || r == nbits - 1) {
        *o++ = (uint8_t)byte;
        byte = 0;
      }
    }
    return;
  }
  if (F.format == 2) {  // "<index>,<weight>,"
    const uint64_t idx = F.index0 + rank[s];
    const int nd = dec_digits(idx);
    uint64_t v = idx;
    for (int i = nd - 1; i >= 0; i--) {
      o[i] = (uint8_t)('0' + v % 10);
      v /= 10;
    }
    o += nd;
    *o++ = ',';
    for (int i = 0; i < F.wlen; i++) *o++ = (uint8_t)F.weight[i];
    *o++ = ',';
  }
  for (int r = 0; r < nbits; r++) *o++ = (uint8_t)('0' + fmt_bit(F, r, s));
  if (F.format == 0 && F.keep_rejected && !fmt_accepted(F, s)) {
    const char* rj = " rejected";
    for (int i = 0; i < 9; i++) *o++ = (uint8_t)rj[i];
  }
  *o = '\n';
}

}  // namespace fs
