// fs_affine.cuh -- host side of the affine frame kernel (frame-only programs, Philox stream).
//
// A frame-only program (k_max = 0: FrameGates, MeasDormantStatic/Random, CondFrame, NoiseBlock,
// Detector/Observable/PostSelect; runtime.py:130-151, :296-330, :546-641) is an affine map over
// GF(2) from (coins, fault indicators) to the output bits: every frame update is an XOR, the
// x<->z swap of MeasDormantRandom and H/SWAP are permutations, and CondFrame XORs a record (itself
// affine) into the frame.  So, per output row r,
//
//     bit_r = const_r  XOR  (XOR of the coins in C_r)  XOR  (XOR over faults f of [r in rows(f)]),
//
// where rows(f) is the set of output rows a single Pauli fault of that case at that site flips
// (its propagation through the rest of the program).  The generator finds const_r, C_r and
// rows(site, case) by propagating one symbolic source per constant / coin / (site, qubit, X|Z)
// element through the program with bitsets, and emits a kernel that never simulates the frame:
//
//   * a pair of warps owns a group of kAffGroup = 8 consecutive 32-shot words (one 32-byte sector
//     of every output row) and a bank-swizzled shared-memory row buffer B[row][8] for them;
//     named barriers (bar.sync id, 64) order the pair's phases;
//   * faults: each warp takes 4 of the words; for one word the 32 lanes evaluate 32 consecutive
//     steps of its noise stream at once (WordFaultGen's process -- the engine stream, so every
//     engine draws the same faults: one Philox block per step, geometric gap
//     floor(ln(U) / log1p(-q)), thinning, case pick), place them with a warp prefix sum of the
//     gaps, and XOR each fault's lane bit into the rows of its case with shared atomics (the
//     case tables live in shared memory when they fit);
//   * coins (Philox, all lanes) and the noiseless (row, coin) terms, XORed in with atomics;
//   * PostSelect / observables in program order (lanes 0..7 of the first warp, one word each),
//     keeping the alive mask of every post-select segment;
//   * copy-out by both warps, 4 rows x 8 words per store: record rows are stored relative to up to
//     kAffMaxParents detector rows (a record's faults are mostly its detectors' faults) and
//     rebuilt here, each row masked with the alive mask in effect at its write.
// Results are bit-identical to the frame interpreter (fs_frame.cuh) and the oracle.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace fsjit {

constexpr int kAffGroup = 8;              // 32-shot words per group (one 32 B sector of every output row)
constexpr int kAffChunk = 32 / kAffGroup;  // rows per copy-out instruction
constexpr int kAffMaxParents = 6;         // rows a copied-out row may be rebuilt from
constexpr int kAffMaxPairs = 16;          // warp pairs per block (one block per SM; named barriers 0..15)
constexpr int kAffDefaultPairs = 14;      // measured best for config 1 (below)
// buffer slot of row r for word wi: r * G + (wi ^ sw(r)), sw(r) = (r / kAffChunk) % G (bank spread)
inline int aff_sw(int r) { return (r / kAffChunk) % kAffGroup; }
constexpr int kAffMaxCoins = 512;         // coin words per 32-shot word (shared memory, 2 KB per word at the limit)
constexpr size_t kAffMaxTerms = 1 << 16;  // coin XOR terms over all rows (code size)

struct AffineKernelSource {
  std::string src;
  std::vector<uint32_t> tables;  // fault tables (case rows, site -> class/case, classes), 16 B sections
  bool tables_smem = false;      // copied into shared memory by every block (else read from HBM/L1)
  int nrows = 0;                 // row-buffer rows per word (+ one zero row)
  int threads = 0;               // block size
  size_t smem = 0;
  std::string why;  // non-empty: not applicable
};

inline AffineKernelSource gen_affine_frame_kernel(const fs_prog_desc& d, const std::vector<int32_t>& ins_all,
                                                  const std::vector<uint32_t>& gates,
                                                  const std::vector<uint32_t>& paulis,
                                                  const std::vector<int32_t>& reclists,
                                                  const std::vector<int32_t>& record_out,
                                                  const std::vector<int32_t>& bit_slot,
                                                  const std::vector<int32_t>& case_pauli_off,
                                                  const std::vector<int32_t>& site_case_off,
                                                  const std::vector<double>& site_prob,
                                                  const std::vector<double>& case_cum, size_t smem_budget) {
  AffineKernelSource K;
  const int n = d.n, R = d.record_count, U = d.num_user_records, D = d.num_detectors, E = d.num_sites;
  (void)bit_slot;
  if (d.k_max != 0) { K.why = "not frame-only"; return K; }
  // ---- rows: user records (col), detectors, one per ObservableIns, hidden bits read by PostSelect
  int n_obs_ins = 0, n_coins = 0;
  std::vector<int> psel_bits;
  for (int i = 0; i < d.num_instrs; i++) {
    const int* I = ins_all.data() + (size_t)i * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]);
    if (op == FS_OP_OBSERVABLE) n_obs_ins++;
    if (op == FS_OP_POSTSELECT) psel_bits.push_back(I[1] == 0 ? R + I[2] : I[2]);
    if (op == FS_OP_MEAS_DRANDOM) n_coins = std::max(n_coins, I[2] + 1);
    if (op != FS_OP_FRAME && op != FS_OP_MEAS_DSTATIC && op != FS_OP_MEAS_DRANDOM && op != FS_OP_COND_FRAME &&
        op != FS_OP_NOISE && op != FS_OP_DETECTOR && op != FS_OP_OBSERVABLE && op != FS_OP_POSTSELECT &&
        op != FS_OP_GAMMA_ROT) {
      K.why = "array instruction";
      return K;
    }
  }
  if (n_coins > kAffMaxCoins) { K.why = "too many coins"; return K; }
  // buffer rows: detectors [0, D), user records [D4, D4 + U), ObservableIns rows from D4 + U4, then
  // hidden bits read by PostSelect (D4, U4 = D, U rounded up to the copy-out chunk: it writes
  // kAffChunk rows of one kind per instruction).  Detectors come first so that record rows can be
  // rebuilt from them (below).
  const int U4 = (U + kAffChunk - 1) / kAffChunk * kAffChunk, D4 = (D + kAffChunk - 1) / kAffChunk * kAffChunk;
  std::vector<int> bit_row(R + D, -1);  // record / detector id -> buffer row
  for (int r = 0; r < R; r++)
    if (record_out[r] >= 0) bit_row[r] = D4 + record_out[r];
  for (int j = 0; j < D; j++) bit_row[R + j] = j;
  int nrows = U4 + D4 + n_obs_ins;
  for (int b : psel_bits)
    if (bit_row[b] < 0) bit_row[b] = nrows++;
  if (nrows >= 8192) { K.why = "too many output rows"; return K; }
  // ---- sources: 0 = constant 1, 1..n_coins = coin ords, then one per (site, qubit, X|Z) element
  const int el0 = 1 + n_coins;
  std::vector<int> site_el0(E + 1, 0);
  std::vector<uint32_t> el_pauli;                   // element -> pauli entry (q << 1 | z)
  std::vector<int> case_el(paulis.size() + 1, -1);  // per pauli entry: element id
  for (int s = 0; s < E; s++) {
    site_el0[s] = (int)el_pauli.size();
    std::map<uint32_t, int> m;
    for (int c = site_case_off[s]; c < site_case_off[s + 1]; c++)
      for (int j = case_pauli_off[c]; j < case_pauli_off[c + 1]; j++) {
        auto it = m.find(paulis[j]);
        if (it == m.end()) {
          it = m.emplace(paulis[j], (int)el_pauli.size()).first;
          el_pauli.push_back(paulis[j]);
        }
        case_el[j] = it->second;
      }
  }
  site_el0[E] = (int)el_pauli.size();
  const size_t NE = el_pauli.size(), NS = el0 + NE, NW = (NS + 63) / 64;
  if ((double)(2 * n + R + D + nrows) * NW * 8 > 2e9) { K.why = "fault-effect table too large"; return K; }
  // ---- symbolic propagation: frame slots and records as bitsets over sources
  std::vector<uint64_t> fr((size_t)2 * n * NW, 0), rec((size_t)(R + D) * NW, 0), rowb((size_t)nrows * NW, 0);
  auto S = [&](int slot) { return fr.data() + (size_t)slot * NW; };
  auto RB = [&](int b) { return rec.data() + (size_t)b * NW; };
  auto xr = [&](uint64_t* a, const uint64_t* b) { for (size_t t = 0; t < NW; t++) a[t] ^= b[t]; };
  auto tog = [&](uint64_t* a, size_t src) { a[src >> 6] ^= 1ull << (src & 63); };
  int obs_row = U4 + D4;
  for (int i = 0; i < d.num_instrs; i++) {
    const int* I = ins_all.data() + (size_t)i * FS_INS_WORDS;
    const bool flip = FS_FLIP(I[0]);
    switch (FS_OPCODE(I[0])) {
      case FS_OP_FRAME:
        for (int j = 0; j < I[2]; j++) {
          const uint32_t g = gates[I[1] + j];
          const int a = FS_GATE_A(g), b = FS_GATE_B(g);
          switch (FS_GATE_G(g)) {
            case FS_G_H: std::swap_ranges(S(a), S(a) + NW, S(n + a)); break;
            case FS_G_S: case FS_G_SDAG: xr(S(n + a), S(a)); break;
            case FS_G_CX: xr(S(b), S(a)); xr(S(n + a), S(n + b)); break;
            case FS_G_CZ: xr(S(n + b), S(a)); xr(S(n + a), S(b)); break;
            case FS_G_SWAP:
              std::swap_ranges(S(a), S(a) + NW, S(b));
              std::swap_ranges(S(n + a), S(n + a) + NW, S(n + b));
              break;
            default: break;
          }
        }
        break;
      case FS_OP_MEAS_DSTATIC:  // record = x ^ flip
        std::copy(S(I[1]), S(I[1]) + NW, RB(I[3]));
        if (flip) tog(RB(I[3]), 0);
        break;
      case FS_OP_MEAS_DRANDOM: {  // record = coin ^ z ^ flip; x' = z ^ coin, z' = x
        const int v = I[1];
        tog(S(n + v), 1 + I[2]);
        std::copy(S(n + v), S(n + v) + NW, RB(I[3]));
        if (flip) tog(RB(I[3]), 0);
        std::swap_ranges(S(v), S(v) + NW, S(n + v));
        break;
      }
      case FS_OP_COND_FRAME:
        for (int j = I[1]; j < I[1] + I[2]; j++) {
          const uint32_t e = paulis[j];
          xr(S(FS_PAULI_Z(e) ? n + FS_PAULI_Q(e) : FS_PAULI_Q(e)), RB(I[3]));
        }
        break;
      case FS_OP_NOISE:
        for (int s = I[1]; s < I[2]; s++)
          for (int el = site_el0[s]; el < site_el0[s + 1]; el++) {
            const uint32_t e = el_pauli[el];
            tog(S(FS_PAULI_Z(e) ? n + FS_PAULI_Q(e) : FS_PAULI_Q(e)), el0 + el);
          }
        break;
      case FS_OP_DETECTOR:
      case FS_OP_OBSERVABLE: {
        std::vector<uint64_t> v(NW, 0);
        for (int j = 0; j < I[3]; j++) xr(v.data(), RB(reclists[I[2] + j]));
        if (FS_OPCODE(I[0]) == FS_OP_DETECTOR) std::copy(v.begin(), v.end(), RB(R + I[1]));
        else std::copy(v.begin(), v.end(), rowb.data() + (size_t)(obs_row++) * NW);
        break;
      }
      default: break;
    }
  }
  for (int b = 0; b < R + D; b++)
    if (bit_row[b] >= 0) std::copy(RB(b), RB(b) + NW, rowb.data() + (size_t)bit_row[b] * NW);
  // ---- sparser rows by differencing: a copied-out record row r may be stored as y_r = v_r ^ v_p1
  // ^ ... for up to kAffMaxParents parent rows (greedy: each round the detector row that most
  // lowers the row's expected fault atomics, sum over cases of P(case) [case flips the row]); the
  // copy-out rebuilds v_r = B[r] ^ B[p1] ^ ... from rows that are never rebuilt themselves, so its
  // chunks carry no shared-memory write-back / re-read chains (FS_AFF_ANY_PARENTS also allows
  // earlier rebuilt rows of the same warp).  For memory experiments the record of ancilla a in round t
  // differs from its round t-1 record by one detector's worth of faults, so record rows shrink
  // to about the size of detector rows.  Rows read before the copy-out (PostSelect, observables)
  // are never differenced.
  std::vector<std::vector<int>> parents(nrows);
  // register parents: record rows rebuilt earlier by the same thread of the copy-out (rows r and q
  // with q = r (mod 8) fall to the same warp of the pair and the same lane row j4), whose rebuilt
  // value is still in a register -- no shared-memory write-back or re-read (a stabilizer's record
  // in round t against its round t-1 record: the residual is one detector's worth of faults)
  std::vector<std::vector<int>> rparents(nrows);
  const bool reg_parents = getenv("FS_AFF_DET_PARENTS") == nullptr && getenv("FS_AFF_ANY_PARENTS") == nullptr;
  auto full_chunk = [&](int q) { return q >= D4 && q < D4 + U && q - q % kAffChunk + kAffChunk <= D4 + U; };
  {
    std::vector<uint8_t> fixed_row(nrows, 0);
    for (int r = U4 + D4; r < nrows; r++) fixed_row[r] = 1;
    for (int b : psel_bits) fixed_row[bit_row[b]] = 1;
    auto el_count = [&](const uint64_t* v) {
      size_t c = 0;
      for (size_t t = 0; t < NW; t++) {
        uint64_t m = v[t];
        if (t * 64 < (size_t)el0) m &= (el0 - t * 64 >= 64) ? 0ull : (~0ull << (el0 - t * 64));
        c += __builtin_popcountll(m);
      }
      return c;
    };
    std::vector<std::vector<int>> orows(NE);  // element -> rows (original vectors)
    std::vector<size_t> sz(nrows);
    for (int r = 0; r < nrows; r++) {
      const uint64_t* v = rowb.data() + (size_t)r * NW;
      sz[r] = el_count(v);
      for (size_t t = 0; t < NW; t++)
        for (uint64_t m = v[t]; m; m &= m - 1) {
          const size_t src = t * 64 + __builtin_ctzll(m);
          if (src >= (size_t)el0) orows[src - el0].push_back(r);
        }
    }
    // cost of a row vector = expected shared atomics it causes: sum over fault cases c of
    // P(case c) [the case flips the row], i.e. of cases with an odd number of the row's elements
    std::vector<std::vector<int>> el_cases(NE);
    std::vector<double> cw(d.num_cases, 0.0);
    for (int st = 0; st < E; st++)
      for (int c = site_case_off[st]; c < site_case_off[st + 1]; c++) {
        cw[c] = case_cum[c] - (c > site_case_off[st] ? case_cum[c - 1] : 0.0);
        if (!(cw[c] > 0.0)) cw[c] = 1e-30;
        for (int j = case_pauli_off[c]; j < case_pauli_off[c + 1]; j++)
          if (case_el[j] >= 0) el_cases[case_el[j]].push_back(c);
      }
    std::vector<uint8_t> cpar(d.num_cases, 0);
    std::vector<int> ctouch;
    auto toggle = [&](const uint64_t* v) {
      for (size_t t = 0; t < NW; t++)
        for (uint64_t m = v[t]; m; m &= m - 1) {
          const size_t src = t * 64 + __builtin_ctzll(m);
          if (src < (size_t)el0) continue;
          for (int c : el_cases[src - el0]) {
            if (!cpar[c]) ctouch.push_back(c);
            cpar[c] ^= 2;  // bit 1 = parity, bit 0 unused (touched list keeps duplicates harmless)
          }
        }
    };
    auto cost2 = [&](const uint64_t* a, const uint64_t* b) {  // cost of a ^ b (b may be null)
      ctouch.clear();
      toggle(a);
      if (b) toggle(b);
      double c = 0.0;
      for (int k : ctouch) {
        if (cpar[k] & 2) c += cw[k];
        cpar[k] = 0;
      }
      return c;
    };
    std::vector<int> ov(nrows, 0);
    std::vector<int> cand;
    int kp = kAffMaxParents;
    // parents among the never-rebuilt rows only (detectors): the copy-out then has no shared-memory
    // write-back / re-read chains between its chunks
    const bool only_fixed = getenv("FS_AFF_ANY_PARENTS") == nullptr;
    if (getenv("FS_AFF_NO_DIFF")) kp = 0;
    if (const char* e = getenv("FS_AFF_PARENTS")) kp = std::max(0, std::min(kAffMaxParents, atoi(e)));
    std::vector<uint64_t> y((size_t)nrows * NW);
    std::copy(rowb.begin(), rowb.end(), y.begin());
    for (int r = 0; r < D4; r++) fixed_row[r] = 1;  // detectors stay as they are (sparse; any warp may read them)
    for (int r = 0; r < nrows; r++) {
      if (fixed_row[r]) continue;
      uint64_t* cur = y.data() + (size_t)r * NW;
      size_t csz = sz[r];
      double ccost = cost2(cur, nullptr);
      for (int round = 0; round < kp && csz > 0; round++) {
        cand.clear();
        for (size_t t = 0; t < NW; t++)
          for (uint64_t m = cur[t]; m; m &= m - 1) {
            const size_t src = t * 64 + __builtin_ctzll(m);
            if (src < (size_t)el0) continue;
            for (int q : orows[src - el0]) {
              if (q >= r - r % kAffChunk) break;
              if (q >= U4 + D4) continue;  // observable / post-select rows: not parents
              const bool regp = reg_parents && !fixed_row[q] && q % (2 * kAffChunk) == r % (2 * kAffChunk) &&
                                full_chunk(q) && r >= D4 && r < D4 + U;
              // a differenced parent must be rebuilt earlier by the same warp of the pair
              if (!fixed_row[q] && !regp && (only_fixed || (q / kAffChunk) % 2 != (r / kAffChunk) % 2)) continue;
              if (ov[q]++ == 0) cand.push_back(q);
            }
          }
        int best = -1;
        size_t bsz = csz;
        double bcost = ccost * (1.0 - 1e-9);
        for (int q : cand) {
          const size_t dsz = csz + sz[q] - 2 * (size_t)ov[q];
          ov[q] = 0;
          if (std::find(parents[r].begin(), parents[r].end(), q) != parents[r].end() ||
              std::find(rparents[r].begin(), rparents[r].end(), q) != rparents[r].end())
            continue;
          const double qc = cost2(cur, rowb.data() + (size_t)q * NW);
          if (qc < bcost) {
            bcost = qc;
            bsz = dsz;
            best = q;
          }
        }
        if (best < 0) break;
        if (reg_parents && !fixed_row[best]) rparents[r].push_back(best);
        else parents[r].push_back(best);
        xr(cur, rowb.data() + (size_t)best * NW);
        csz = bsz;
        ccost = bcost;
      }
    }
    rowb.swap(y);
  }
  // ---- transpose: element -> rows; case -> XOR of its elements' rows
  std::vector<std::vector<uint16_t>> el_rows(NE);
  for (int r = 0; r < nrows; r++) {
    const uint64_t* v = rowb.data() + (size_t)r * NW;
    for (size_t t = 0; t < NW; t++)
      for (uint64_t m = v[t]; m; m &= m - 1) {
        const size_t src = t * 64 + __builtin_ctzll(m);
        if (src >= (size_t)el0) el_rows[src - el0].push_back((uint16_t)r);
      }
  }
  std::vector<uint32_t> crow_off(d.num_cases + 1, 0);
  std::vector<uint16_t> crows;
  std::vector<uint8_t> par(nrows, 0);
  std::vector<uint16_t> touched;
  for (int c = 0; c < d.num_cases; c++) {
    crow_off[c] = (uint32_t)crows.size();
    touched.clear();
    for (int j = case_pauli_off[c]; j < case_pauli_off[c + 1]; j++) {
      if (case_el[j] < 0) continue;
      for (uint16_t r : el_rows[case_el[j]]) {
        touched.push_back(r);
        par[r] ^= 1;
      }
    }
    std::sort(touched.begin(), touched.end());
    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
    for (uint16_t r : touched) {  // stored as the row's buffer slot for word 0: slot(r, wi) = e ^ wi
      if (par[r]) crows.push_back((uint16_t)(r * kAffGroup | aff_sw(r)));
      par[r] = 0;
    }
  }
  crow_off[d.num_cases] = (uint32_t)crows.size();
  // ---- site classes: sites with identical (p, case_cum) share one entry of the case-pick table
  int cw = 1;  // case_cum width per class
  for (int st = 0; st < E; st++) cw = std::max(cw, site_case_off[st + 1] - site_case_off[st]);
  std::map<std::vector<uint64_t>, int> cls_of;
  std::vector<std::vector<double>> cls_cum;
  std::vector<double> cls_prob;
  std::vector<int32_t> cls_nc;
  std::vector<uint16_t> site_cls(E);
  for (int st = 0; st < E; st++) {
    std::vector<uint64_t> key;
    auto bits = [](double v) { uint64_t u; memcpy(&u, &v, 8); return u; };
    key.push_back(bits(site_prob[st]));
    for (int c = site_case_off[st]; c < site_case_off[st + 1]; c++) key.push_back(bits(case_cum[c]));
    auto it = cls_of.find(key);
    if (it == cls_of.end()) {
      it = cls_of.emplace(key, (int)cls_prob.size()).first;
      cls_prob.push_back(site_prob[st]);
      cls_nc.push_back(site_case_off[st + 1] - site_case_off[st]);
      std::vector<double> cc(cw, 0.0);
      for (int c = site_case_off[st]; c < site_case_off[st + 1]; c++) cc[c - site_case_off[st]] = case_cum[c];
      cls_cum.push_back(cc);
    }
    site_cls[st] = (uint16_t)it->second;
  }
  if (cls_prob.size() >= 65535) { K.why = "too many site classes"; return K; }
  const int ncls = (int)cls_prob.size();
  // ---- table blob (u32 words, 16 B sections): crows u16 | crow_off u16 or u32 | site_case u32 |
  // site_cls u16 | cls_nc i32 | cls_prob f64 | cls_cum f64 [ncls][cw]
  const bool off16 = crows.size() < 65536;
  auto& T = K.tables;
  auto sec = [&](size_t bytes) {
    size_t w = T.size();
    T.resize(w + ((bytes + 15) / 16) * 4 + 4, 0u);  // +16 B keeps empty sections distinct
    return w;
  };
  const size_t o_crows = sec(crows.size() * 2);
  memcpy(T.data() + o_crows, crows.data(), crows.size() * 2);
  const size_t o_coff = sec(crow_off.size() * (off16 ? 2 : 4));
  if (off16) {
    std::vector<uint16_t> c16(crow_off.begin(), crow_off.end());
    memcpy(T.data() + o_coff, c16.data(), c16.size() * 2);
  } else {
    memcpy(T.data() + o_coff, crow_off.data(), crow_off.size() * 4);
  }
  const size_t o_scase = sec((size_t)E * 4);
  if (E) memcpy(T.data() + o_scase, site_case_off.data(), (size_t)E * 4);
  const size_t o_scls = sec((size_t)E * 2);
  if (E) memcpy(T.data() + o_scls, site_cls.data(), (size_t)E * 2);
  const size_t o_cnc = sec((size_t)ncls * 4);
  if (ncls) memcpy(T.data() + o_cnc, cls_nc.data(), (size_t)ncls * 4);
  const size_t o_cp = sec((size_t)ncls * 8);
  if (ncls) memcpy(T.data() + o_cp, cls_prob.data(), (size_t)ncls * 8);
  const size_t o_cc = sec((size_t)ncls * cw * 8);
  for (int c = 0; c < ncls; c++) memcpy(T.data() + o_cc + (size_t)c * cw * 2, cls_cum[c].data(), (size_t)cw * 8);
  const size_t o_cs = sec((size_t)ncls * 8);
  for (int c = 0; c < ncls; c++) {
    const double sc = cls_prob[c] > 0.0 ? (double)cls_nc[c] / cls_prob[c] : 0.0;
    memcpy(T.data() + o_cs + 2 * c, &sc, 8);
  }
  // copy-out side tables: parent slot of every row (the zero row when not differenced), its
  // post-select segment (alive mask in effect at its write), noiseless terms (row slot, coin word;
  // coin n_coins = the all-ones word of a constant)
  const int zrow = nrows;
  std::vector<int> row_seg(nrows + 1, 0);
  int npsel = 0;
  for (int i = 0; i < d.num_instrs; i++) {
    const int* I = ins_all.data() + (size_t)i * FS_INS_WORDS;
    switch (FS_OPCODE(I[0])) {
      case FS_OP_MEAS_DSTATIC:
      case FS_OP_MEAS_DRANDOM:
        if (record_out[I[3]] >= 0) row_seg[bit_row[I[3]]] = npsel;
        break;
      case FS_OP_DETECTOR: row_seg[bit_row[R + I[1]]] = npsel; break;
      case FS_OP_POSTSELECT: npsel++; break;
      default: break;
    }
  }
  size_t o_ps[kAffMaxParents];
  for (int k = 0; k < kAffMaxParents; k++) {
    o_ps[k] = sec((size_t)(nrows + 1) * 2);
    std::vector<uint16_t> ps(nrows + 1);
    for (int r = 0; r <= nrows; r++) {
      const int pr = r < nrows && (int)parents[r].size() > k ? parents[r][k] : zrow;
      ps[r] = (uint16_t)(pr * kAffGroup | aff_sw(pr));
    }
    memcpy(T.data() + o_ps[k], ps.data(), ps.size() * 2);
  }
  const size_t o_seg = sec((size_t)(nrows + 1) * 2);
  {
    std::vector<uint16_t> sg(row_seg.begin(), row_seg.end());
    memcpy(T.data() + o_seg, sg.data(), sg.size() * 2);
  }
  std::vector<uint32_t> terms_tab;  // slot0 | coin << 16
  for (int r = 0; r < nrows; r++) {
    const uint64_t* v = rowb.data() + (size_t)r * NW;
    const uint32_t sl = (uint32_t)(r * kAffGroup | aff_sw(r));
    if (v[0] & 1ull) terms_tab.push_back(sl | (uint32_t)n_coins << 16);
    for (int c = 0; c < n_coins; c++)
      if ((v[(1 + c) >> 6] >> ((1 + c) & 63)) & 1ull) terms_tab.push_back(sl | (uint32_t)c << 16);
  }
  // coin-major order: the 4 terms one warp instruction applies then hit distinct rows (a row's
  // coins are consecutive in row-major order and would collide on one shared word)
  std::stable_sort(terms_tab.begin(), terms_tab.end(), [](uint32_t a, uint32_t b) { return (a >> 16) < (b >> 16); });
  if (terms_tab.size() > kAffMaxTerms) { K.why = "noiseless part too large"; return K; }
  const size_t o_terms = sec(terms_tab.size() * 4);
  if (!terms_tab.empty()) memcpy(T.data() + o_terms, terms_tab.data(), terms_tab.size() * 4);
  const size_t o_ln = sec(FS_LN_TAB_ENTRIES * 16);
  {
    static const double lt[FS_LN_TAB_ENTRIES][2] = FS_LN_TAB_INIT;
    memcpy(T.data() + o_ln, lt, sizeof lt);
  }
  const size_t tbl_bytes = T.size() * 4;
  // ---- launch shape: a pair of warps per 8-word group; per pair a row buffer (+ a zero row),
  // the alive masks of the post-select segments and the group's coin words
  K.nrows = (nrows + 1 + 3) / 4 * 4;  // + zero row, padded so the 32 dump words start at a multiple of 32
  const int nblk = (n_coins + 3) / 4, cstride = (n_coins + 1) | 1;  // coin words + all-ones word (odd stride)
  const size_t per_pair =
      ((size_t)K.nrows + psel_bits.size() + 1) * kAffGroup * 4 + 32 * 4 + (size_t)kAffGroup * cstride * 4;
  int npairs = 0;
  {
    // at most 14 pairs by default: config 1 measured 0.198 ms at 14 pairs (28 warps / SM), 0.201 at
    // 16 and 0.206 at 12 (FS_AFF_PAIRS overrides, up to kAffMaxPairs)
    const char* ep = getenv("FS_AFF_PAIRS");
    const size_t cap = ep ? (size_t)std::max(1, std::min(kAffMaxPairs, atoi(ep))) : (size_t)kAffDefaultPairs;
    npairs = (int)std::min<size_t>(cap, tbl_bytes < smem_budget ? (smem_budget - tbl_bytes) / per_pair : 0);
    K.tables_smem = npairs >= 4 && !getenv("FS_AFF_GLOBAL_TABLES");
    if (!K.tables_smem) npairs = (int)std::min<size_t>(cap, smem_budget / per_pair);
    if (npairs < 1) { K.why = "row buffer does not fit shared memory"; return K; }
    // an even pair count puts the same number of warps on each of the SM's four schedulers (the
    // kernel is issue-bound: 15 pairs = 8/8/7/7 warps ran slower than 14 pairs = 7/7/7/7)
    if (npairs > 1 && !ep) npairs &= ~1;
    K.threads = npairs * 64;
    K.smem = per_pair * npairs + (K.tables_smem ? tbl_bytes : 0);
  }
  if (getenv("FS_AFF_VERBOSE")) {
    std::vector<int> hist(34, 0);
    for (int c = 0; c < d.num_cases; c++) hist[std::min<uint32_t>(33, crow_off[c + 1] - crow_off[c])]++;
    fprintf(stderr, "aff: case row-count histogram:");
    for (int h = 0; h < 34; h++) if (hist[h]) fprintf(stderr, " %d:%d", h, hist[h]);
    fprintf(stderr, "\n");
    size_t el_total = 0;
    for (auto& v : el_rows) el_total += v.size();
    {
      std::vector<int> hit(nrows, 0), npar(kAffMaxParents + 1, 0);
      for (auto& v : el_rows)
        for (int r : v) hit[r] = 1;
      int nhit = 0, nhit_det = 0;
      for (int r = 0; r < nrows; r++) { nhit += hit[r]; if (r < D4) nhit_det += hit[r]; }
      for (int r = 0; r < nrows; r++) npar[std::min<size_t>(kAffMaxParents, parents[r].size() + rparents[r].size())]++;
      int nreg = 0;
      for (int r = 0; r < nrows; r++) nreg += (int)rparents[r].size();
      fprintf(stderr, "aff: register parents %d\n", nreg);
      fprintf(stderr, "aff: rows with fault residual %d (detector rows %d of %d); parents histogram:", nhit, nhit_det, D);
      for (int k = 0; k <= kAffMaxParents; k++) fprintf(stderr, " %d:%d", k, npar[k]);
      fprintf(stderr, "\n");
    }
    fprintf(stderr,
            "aff: rows %d coins %d elements %zu element-rows %zu cases %d case-rows %zu classes %d tables %zu B "
            "(%s) warps %d\n",
            nrows, n_coins, NE, el_total, d.num_cases, crows.size(), ncls, tbl_bytes,
            K.tables_smem ? "smem" : "global", K.threads / 32);
  }

  // ---- kernel source
  // phase 1 (all lanes): zero the group's row buffer, XOR in the faults of its 8 words
  // phase 2 (lanes 0..7, lane = word): XOR the noiseless part (constant ^ coins) into the rows
  //   that have one, evaluate PostSelect / observables in program order, keep the alive mask of
  //   every post-select segment in AL[seg][word]
  // phase 3 (all lanes, lane = (row & 3, word)): copy rows out, 4 rows x 8 words (four 32 B
  //   sectors) per instruction, each masked with the alive mask in effect at its write
  const int G = kAffGroup;
  std::ostringstream p2;
  {
    int seg = 0;
    obs_row = U4 + D4;
    for (int i = 0; i < d.num_instrs; i++) {
      const int* I = ins_all.data() + (size_t)i * FS_INS_WORDS;
      switch (FS_OPCODE(I[0])) {
        case FS_OP_OBSERVABLE: {
          const int row = obs_row++;
          p2 << "      ob" << I[1] << " ^= B[" << row * G << " + (lane ^ " << aff_sw(row) << ")] & alive;\n";
          break;
        }
        case FS_OP_POSTSELECT: {
          const int bid = I[1] == 0 ? R + I[2] : I[2];
          const int row = bit_row[bid];
          p2 << "      alive &= ~((B[" << row * G << " + (lane ^ " << aff_sw(row) << ")]" << (I[3] ? " ^ 0xFFFFFFFFu" : "")
             << ") & alive);\n";
          p2 << "      AL[" << (seg + 1) * G << " + lane] = alive;\n";
          seg++;
          break;
        }
        default: break;
      }
    }
  }
  std::ostringstream o;
  if (const char* dg = getenv("FS_AFF_DIAG")) o << "#define FS_AFF_DIAG " << atoi(dg) << "\n";  // profiling only
  if (getenv("FS_AFF_BALANCED")) o << "#define FS_AFF_ROWS aff_rows_bal\n";  // A/B: load-balanced row loop
  if (!getenv("FS_AFF_CLS_TABLES")) {
    if (ncls <= 4) {  // class probabilities, case counts and scales as constants (no table loads)
      o << "#define FS_AFF_CLS_CONST 1\n";
      if (!getenv("FS_AFF_NO_SAFEZONE")) {
        // eps(k) > max_i |cum[i] * nc / p - (i + 1)| (+ margin for the rounding of x * nc / p): a
        // y = x * nc / p at least eps from every integer has floor(y) == bisect_right(cum, x)
        o << "#define FS_AFF_SAFEZONE 1\n";
        o << "__device__ __forceinline__ double fs_aff_cls_eps(int k) { return ";
        for (int c = 0; c < ncls; c++) {
          const double sc = cls_prob[c] > 0.0 ? (double)cls_nc[c] / cls_prob[c] : 0.0;
          double e = 0.0;
          for (int i = 0; i + 1 < cls_nc[c]; i++) e = std::max(e, std::fabs(cls_cum[c][i] * sc - (i + 1)));
          e = e * 2.0 + 1e-9;
          if (!(e < 0.25)) e = 2.0;  // not near-uniform: always the exact path
          if (c + 1 < ncls) o << "k == " << c << " ? " << hexd(e) << " : ";
          else o << hexd(e);
        }
        if (ncls == 0) o << "2.0";
        o << "; }\n";
      }
      o << "__device__ __forceinline__ int fs_aff_cls_nc(int k) { return ";
      for (int c = 0; c + 1 < ncls; c++) o << "k == " << c << " ? " << cls_nc[c] << " : ";
      o << (ncls ? cls_nc[ncls - 1] : 0) << "; }\n";
      o << "__device__ __forceinline__ double fs_aff_cls_prob(int k) { return ";
      for (int c = 0; c + 1 < ncls; c++) o << "k == " << c << " ? " << hexd(cls_prob[c]) << " : ";
      o << hexd(ncls ? cls_prob[ncls - 1] : 0.0) << "; }\n";
      o << "__device__ __forceinline__ double fs_aff_cls_scale(int k) { return ";
      for (int c = 0; c + 1 < ncls; c++) {
        const double sc = cls_prob[c] > 0.0 ? (double)cls_nc[c] / cls_prob[c] : 0.0;
        o << "k == " << c << " ? " << hexd(sc) << " : ";
      }
      {
        const double sc = ncls && cls_prob[ncls - 1] > 0.0 ? (double)cls_nc[ncls - 1] / cls_prob[ncls - 1] : 0.0;
        o << hexd(sc) << "; }\n";
      }
    }
  }
  o << "#include \"fs_jit_kernels.cuh\"\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << K.threads << ", 1) fs_aff_frame(fs::DevProg P, fs::RunArgs A, "
       "const uint32_t* __restrict__ tbl) {\n";
  o << "  extern __shared__ __align__(16) uint32_t smem[];\n";
  o << "  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;\n";
  size_t bufw = 0;
  if (K.tables_smem) {
    bufw = T.size();
    o << "  for (int i = threadIdx.x; i < " << T.size() / 4 << "; i += " << K.threads
      << ") reinterpret_cast<uint4*>(smem)[i] = __ldg(reinterpret_cast<const uint4*>(tbl) + i);\n";
    o << "  __syncthreads();\n";
    o << "  const uint32_t* const tb = smem;\n";
  } else {
    o << "  const uint32_t* const tb = tbl;\n";
  }
  o << "  fs::AffTabs<" << (off16 ? "true" : "false") << "> tabs;\n";
  o << "  tabs.crows = reinterpret_cast<const uint16_t*>(tb + " << o_crows << ");\n";
  o << "  tabs.crow_off = tb + " << o_coff << ";\n";
  o << "  tabs.site_case = tb + " << o_scase << ";\n";
  o << "  tabs.site_cls = reinterpret_cast<const uint16_t*>(tb + " << o_scls << ");\n";
  o << "  tabs.cls_nc = reinterpret_cast<const int*>(tb + " << o_cnc << ");\n";
  o << "  tabs.cls_prob = reinterpret_cast<const double*>(tb + " << o_cp << ");\n";
  o << "  tabs.cls_cum = reinterpret_cast<const double*>(tb + " << o_cc << ");\n";
  o << "  tabs.lntab = reinterpret_cast<const double2*>(tb + " << o_ln << ");\n";
  o << "  tabs.cls_scale = reinterpret_cast<const double*>(tb + " << o_cs << ");\n";
  o << "  tabs.cw = " << cw << ";\n";
  for (int k = 0; k < kAffMaxParents; k++)
    o << "  const uint16_t* const PS" << k << " = reinterpret_cast<const uint16_t*>(tb + " << o_ps[k] << ");\n";
  o << "  const uint16_t* const SEG = reinterpret_cast<const uint16_t*>(tb + " << o_seg << ");\n";
  o << "  const uint32_t* const TERMS = tb + " << o_terms << ";\n";
  (void)o_seg;
  o << "  const int pair = wib >> 1, half = wib & 1, t64 = threadIdx.x & 63;\n";
  o << "  uint32_t* const B = smem + " << bufw << " + pair * " << (size_t)K.nrows * G + 32 << ";\n";
  o << "  tabs.dump = " << (size_t)K.nrows * G << ";\n";
  const size_t bufs = (size_t)npairs * ((size_t)K.nrows * G + 32);
  o << "  uint32_t* const AL = smem + " << bufw + bufs << " + pair * " << (npsel + 1) * G << ";\n";
  o << "  uint32_t* const CW = smem + " << bufw + bufs + (size_t)npairs * (npsel + 1) * G << " + pair * " << G * cstride
    << ";\n";
  o << "  const uint64_t word0 = A.shot0 >> 5;\n  const uint64_t seed = A.seed;\n";
  o << "  const uint32_t ngroups = (A.W + " << G - 1 << ") / " << G << ";\n";
  o << "  const int j4 = lane / " << G << ", wi = lane % " << G << ";\n";
  o << "  if (t64 < " << G << ") CW[t64 * " << cstride << " + " << n_coins << "] = 0xFFFFFFFFu;\n";
  o << "  for (uint32_t grp = blockIdx.x * " << npairs << " + pair; grp < ngroups; grp += gridDim.x * " << npairs << ") {\n";
  o << "    for (int i = t64; i < " << (size_t)K.nrows * G / 4
    << "; i += 64) reinterpret_cast<uint4*>(B)[i] = make_uint4(0u, 0u, 0u, 0u);\n";
  o << "    fs::pair_sync(pair);\n";
  // uniform classes: every cum[i] within (i, i + 2) bins of the grid i * p / nc, with margin for rounding
  bool uniform = true;
  for (int c = 0; c < ncls; c++) {
    const double sc = cls_prob[c] > 0.0 ? (double)cls_nc[c] / cls_prob[c] : 0.0;
    for (int i = 0; i + 1 < cls_nc[c]; i++) {
      const double gpos = cls_cum[c][i] * sc;  // ideal i + 1
      if (!(std::fabs(gpos - (i + 1)) < 0.25)) uniform = false;
    }
  }
  if (getenv("FS_AFF_NONUNIFORM")) uniform = false;
  o << "    fs::aff_group_faults<" << G << ", " << (off16 ? "true" : "false") << ", " << (uniform ? "true" : "false")
    << ">(P, tabs, B, seed, word0, grp, A.W, lane, half * " << G / 2 << ", half * " << G / 2 << " + " << G / 2 << ");\n";
  if (n_coins > 0) {  // coin blocks of the warp's 4 words: lane = (block % 8, word)
    o << "    for (int cb = lane >> 2; cb < " << nblk << "; cb += 8) {\n";
    o << "      const int cw_ = half * " << G / 2 << " + (lane & 3);\n";
    o << "      const uint4 v = fs::coin_block(seed, word0 + grp * " << G << " + cw_, cb);\n";
    o << "      uint32_t* const d = CW + cw_ * " << cstride << " + cb * 4;\n";
    o << "      d[0] = v.x;";
    o << " if (cb * 4 + 1 < " << n_coins << ") d[1] = v.y;";
    o << " if (cb * 4 + 2 < " << n_coins << ") d[2] = v.z;";
    o << " if (cb * 4 + 3 < " << n_coins << ") d[3] = v.w;\n";
    o << "    }\n";
  }
  o << "    fs::pair_sync(pair);\n";
  if (!terms_tab.empty()) {
    o << "    for (int t = j4 + half * " << kAffChunk << "; t < " << terms_tab.size() << "; t += " << 2 * kAffChunk << ") {\n";
    o << "      const uint32_t e = TERMS[t];\n";
    o << "      atomicXor(B + ((e & 0xFFFFu) ^ wi), CW[wi * " << cstride << " + (e >> 16)]);\n";
    o << "    }\n    fs::pair_sync(pair);\n";
  }
  o << "    if (half == 0 && lane < " << G << ") {\n";
  o << "      const uint32_t w = grp * " << G << " + lane;\n";
  o << "      const uint64_t nleft = w < A.W ? A.nshots - (uint64_t)w * 32 : 0;\n";
  o << "      const uint32_t valid = nleft >= 32 ? 0xFFFFFFFFu : ((1u << nleft) - 1u);\n";
  o << "      uint32_t alive = valid;\n";
  o << "      AL[lane] = valid;\n";
  for (int jj = 0; jj < d.num_observables; jj++) o << "      uint32_t ob" << jj << " = 0u;\n";
  o << p2.str();
  o << "      if (w < A.W) {\n";
  for (int jj = 0; jj < d.num_observables; jj++)
    o << "        A.obs[(size_t)" << jj << " * A.ostride + w] = ob" << jj << " & valid;\n";
  o << "        A.accepted[w] = alive & valid;\n        A.error[w] = 0u;\n      }\n";
  o << "    }\n";
  o << "    fs::pair_sync(pair);\n";
  o << "    {\n";
  o << "      const uint32_t w = grp * " << G << " + wi;\n";
  o << "      if (w < A.W) {\n";
  if (npsel == 0) o << "        const uint32_t m0 = AL[wi];\n";
  o << "        uint32_t* const mo = A.meas + (size_t)j4 * A.ostride + w;\n";
  o << "        uint32_t* const dout = A.det + (size_t)j4 * A.ostride + w;\n";
  o << "        const size_t sc = (size_t)" << kAffChunk << " * A.ostride;\n";
  std::vector<uint8_t> is_parent(nrows + 1, 0), is_rparent(nrows + 1, 0);
  for (int r = 0; r < nrows; r++) {
    for (int q : parents[r]) is_parent[q] = 1;
    for (int q : rparents[r]) is_rparent[q] = 1;
  }
  int cur_half = 0;
  auto emit_copy = [&](int r0, int cnt, const char* base, int rbase) {
    const int RC = kAffChunk;
    for (int r = r0; r < r0 + cnt; r += RC) {
      if (r / RC % 2 != cur_half) continue;  // the other warp of the pair copies this chunk
      // rows r..r+RC-1 (r a multiple of RC): lane row r + j4 at slot (r + j4) * G + (wi ^ sw(r)); a
      // differenced row adds its (already rebuilt) parents and is written back for later children
      const int rem = std::min(RC, r0 + cnt - r);
      size_t np = 0;
      for (int q = 0; q < rem; q++) np = std::max(np, parents[r + q].size());
      const std::string m = npsel == 0 ? "m0" : "AL[SEG[" + std::to_string(r) + " + j4] * " + std::to_string(G) + " + wi]";
      // a full chunk some later row uses as a register parent keeps its value in v<r>
      bool rkeep = false;
      for (int q = 0; q < rem && !rkeep; q++) rkeep = is_rparent[r + q];
      const std::string V = rkeep ? "v" + std::to_string(r) : std::string("v");
      o << "        ";
      if (!rkeep) o << "{";
      if (rem < RC) o << " if (j4 < " << rem << ") {";
      o << " uint32_t " << V << " = B[" << r * G << " + j4 * " << G << " + (wi ^ " << aff_sw(r) << ")];";
      size_t nr = 0;
      for (int q = 0; q < rem; q++) nr = std::max(nr, rparents[r + q].size());
      for (size_t k = 0; k < nr; k++) {
        const int p0 = rparents[r].size() > k ? rparents[r][k] : -1;
        bool same = rem == RC && p0 >= 0 && p0 % RC == 0;
        for (int q = 1; q < rem && same; q++) same = rparents[r + q].size() > k && rparents[r + q][k] == p0 + q;
        if (same) {
          o << " " << V << " ^= v" << p0 << ";";
        } else {  // lane row j4 = q holds row p of chunk p - q (p = r + q mod 8)
          o << " " << V << " ^= ";
          for (int q = 0; q < rem; q++) {
            const std::string x = rparents[r + q].size() > k ? "v" + std::to_string(rparents[r + q][k] - q) : "0u";
            if (q + 1 < rem) o << "j4 == " << q << " ? " << x << " : ";
            else o << x;
          }
          o << ";";
        }
      }
      for (size_t k = 0; k < np; k++) {
        // parents of the chunk's rows at one common offset from a chunk-aligned row: constant slots
        const int p0 = parents[r].size() > k ? parents[r][k] : -1;
        bool same = p0 >= 0 && p0 % RC == 0;
        for (int q = 1; q < rem && same; q++) same = parents[r + q].size() > k && parents[r + q][k] == p0 + q;
        if (same) {
          o << " " << V << " ^= B[" << p0 * G << " + j4 * " << G << " + (wi ^ " << aff_sw(p0) << ")];";
        } else {
          o << " " << V << " ^= B[PS" << k << "[" << r << " + j4] ^ wi];";
        }
      }
      bool wb = false;  // some later row rebuilds from one of these rows
      for (int q = 0; q < rem && !wb; q++) wb = is_parent[r + q];
      if ((np || nr) && wb) o << " B[" << r * G << " + j4 * " << G << " + (wi ^ " << aff_sw(r) << ")] = " << V << ";";
      o << " " << base << "[" << (r - rbase) / RC << " * sc] = " << V << " & " << m << ";";
      if (rem < RC) o << " }";
      if (!rkeep) o << " }";
      o << "\n";
    }
  };
  const int diag = getenv("FS_AFF_DIAG") ? atoi(getenv("FS_AFF_DIAG")) : 0;  // profiling only
  for (cur_half = 0; cur_half < 2; cur_half++) {
    o << "        " << (cur_half == 0 ? "if (half == 0) {" : "} else {") << "\n";
    if (diag != 4 && diag != 6) {
      emit_copy(0, D, "dout", 0);
      emit_copy(D4, U, "mo", D4);
    }
  }
  o << "        }\n";
  o << "      }\n    }\n";
  o << "    fs::pair_sync(pair);\n  }\n}\n";
  K.src = o.str();
  return K;
}

}  // namespace fsjit
