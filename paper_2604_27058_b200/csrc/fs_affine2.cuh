// fs_affine2.cuh -- host side of the lane-per-word affine frame kernel (frame-only programs,
// Philox stream): the config-1 kernel.
//
// Same affine decomposition as fs_affine.cuh (every output bit = const ^ coins ^ fault effects,
// runtime.py:130-151, :296-330, :546-641), organised for the shared-memory / MIO pipe, which binds
// the warp-pair kernel (profiles/r2_c1_aff_ncu.md: shared atomics, row-list loads, shuffles and
// stores of one SM share it):
//
//   * lane = one 32-shot word; a warp owns 32 consecutive words (1024 shots) and a column-private
//     row buffer B[row][32] in shared memory (bank = lane): fault rows are XORed with plain
//     load / store pairs, no atomics, no bank conflicts;
//   * each lane runs its word's noise stream sequentially -- exactly WordFaultGen's process (the
//     same Philox block per step, gap, thinning and case as every other engine) -- and queues its
//     faults (case, shot bit) in shared memory; the queue is then applied per row pass, a lane
//     walking its own queue (no cross-lane work: no shuffles, no scans);
//   * the output is emitted as straight-line code in PROGRAM ORDER, uniform across lanes: each
//     value (user record, detector, observable update, post-selected bit) is rebuilt as
//     B[row] ^ (earlier values, in registers) ^ (coin words, in registers) ^ const, stored with one
//     coalesced 128-byte store per row, masked by the alive mask in effect at its write
//     (PostSelect, runtime.py:632-641, updates the mask in the same program order);
//   * earlier values serve as parents (chains such as record(a, t) = detector(a, t) ^ record(a, t-1)
//     leave no fault residual at all), so only values with a residual own a buffer row; rows are
//     split into passes when the buffer for all of them would cost occupancy.
// Bit-identical to fs_affine.cuh, the frame interpreter and the oracle.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace fsjit {

constexpr int kAff2MaxCoins = 64;     // coin words per lane live in registers
constexpr int kAff2MaxParents = 6;
constexpr int kAff2MaxItems = 4096;

struct Affine2KernelSource {
  std::string src;
  std::vector<uint32_t> tables;
  int threads = 0;   // block size (warps x 32), one block per SM
  size_t smem = 0;
  int npass = 0, nbp = 0, qcap = 0, nbuf = 0, nitems = 0;
  size_t ovf_per_lane = 0;  // queue entries beyond qcap spill to global memory (ovf)
  std::string why;          // non-empty: not applicable (fs_affine.cuh is used)
};

inline Affine2KernelSource gen_affine2_kernel(const fs_prog_desc& d, const std::vector<int32_t>& ins_all,
                                              const std::vector<uint32_t>& gates, const std::vector<uint32_t>& paulis,
                                              const std::vector<int32_t>& reclists,
                                              const std::vector<int32_t>& record_out,
                                              const std::vector<int32_t>& case_pauli_off,
                                              const std::vector<int32_t>& site_case_off,
                                              const std::vector<double>& site_prob,
                                              const std::vector<double>& case_cum, int num_runs, size_t smem_budget) {
  Affine2KernelSource K;
  const int n = d.n, R = d.record_count, D = d.num_detectors, E = d.num_sites;
  if (d.k_max != 0) { K.why = "not frame-only"; return K; }
  int n_coins = 0;
  for (int i = 0; i < d.num_instrs; i++) {
    const int* I = ins_all.data() + (size_t)i * FS_INS_WORDS;
    const int op = FS_OPCODE(I[0]);
    if (op == FS_OP_MEAS_DRANDOM) n_coins = std::max(n_coins, I[2] + 1);
    if (op != FS_OP_FRAME && op != FS_OP_MEAS_DSTATIC && op != FS_OP_MEAS_DRANDOM && op != FS_OP_COND_FRAME &&
        op != FS_OP_NOISE && op != FS_OP_DETECTOR && op != FS_OP_OBSERVABLE && op != FS_OP_POSTSELECT &&
        op != FS_OP_GAMMA_ROT) {
      K.why = "array instruction";
      return K;
    }
  }
  if (n_coins > kAff2MaxCoins) { K.why = "too many coins for registers"; return K; }
  // ---- sources: 0 = constant 1, 1..n_coins = coin ords, then one per (site, qubit, X|Z) element
  const int el0 = 1 + n_coins;
  std::vector<int> site_el0(E + 1, 0);
  std::vector<uint32_t> el_pauli;
  std::vector<int> case_el(paulis.size() + 1, -1);
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
  if ((double)(2 * n + R + D + 64) * NW * 8 > 2e9) { K.why = "fault-effect table too large"; return K; }
  // ---- symbolic propagation (frame slots and records as bitsets over the sources)
  std::vector<uint64_t> fr((size_t)2 * n * NW, 0), rec((size_t)(R + D) * NW, 0);
  auto S = [&](int slot) { return fr.data() + (size_t)slot * NW; };
  auto RB = [&](int b) { return rec.data() + (size_t)b * NW; };
  auto xr = [&](uint64_t* a, const uint64_t* b) { for (size_t t = 0; t < NW; t++) a[t] ^= b[t]; };
  auto tog = [&](uint64_t* a, size_t src) { a[src >> 6] ^= 1ull << (src & 63); };
  // items in program order: 0 record (user), 1 detector, 2 observable update, 3 post-select
  struct Item { int kind, idx, req, ref; std::vector<uint64_t> v; };
  std::vector<Item> items;
  std::vector<int> item_of_bit(R + D, -1);  // record / detector id -> item holding its value
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
      case FS_OP_MEAS_DSTATIC:
      case FS_OP_MEAS_DRANDOM: {
        const int v = I[1], r = I[3];
        if (FS_OPCODE(I[0]) == FS_OP_MEAS_DSTATIC) {
          std::copy(S(v), S(v) + NW, RB(r));
        } else {  // record = coin ^ z ^ flip; x' = z ^ coin, z' = x
          tog(S(n + v), 1 + I[2]);
          std::copy(S(n + v), S(n + v) + NW, RB(r));
          std::swap_ranges(S(v), S(v) + NW, S(n + v));
        }
        if (flip) tog(RB(r), 0);
        if (record_out[r] >= 0) {
          items.push_back({0, record_out[r], 0, r, std::vector<uint64_t>(RB(r), RB(r) + NW)});
          item_of_bit[r] = (int)items.size() - 1;
        }
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
        if (FS_OPCODE(I[0]) == FS_OP_DETECTOR) {
          std::copy(v.begin(), v.end(), RB(R + I[1]));
          items.push_back({1, I[1], 0, R + I[1], v});
          item_of_bit[R + I[1]] = (int)items.size() - 1;
        } else {
          items.push_back({2, I[1], 0, -1, v});
        }
        break;
      }
      case FS_OP_POSTSELECT: {
        const int bid = I[1] == 0 ? R + I[2] : I[2];
        if (item_of_bit[bid] < 0) {  // a hidden record read by PostSelect: its own (unstored) item
          items.push_back({4, -1, 0, bid, std::vector<uint64_t>(RB(bid), RB(bid) + NW)});
          item_of_bit[bid] = (int)items.size() - 1;
        }
        items.push_back({3, item_of_bit[bid], I[3], bid, {}});
        break;
      }
      default: break;
    }
  }
  const int NI = (int)items.size();
  if (NI > kAff2MaxItems) { K.why = "too many output values"; return K; }
  // computation order: the alive mask only changes at PostSelect, so inside each post-select
  // segment values may be computed in any order -- detectors first, so that records and
  // observables can be rebuilt from them (a detector is the XOR of a few records; its fault
  // support is the sparse one)
  std::vector<int> order;
  for (int b = 0; b < NI;) {
    int e = b;
    while (e < NI && items[e].kind != 3) e++;
    for (int q = b; q < e; q++) if (items[q].kind == 1) order.push_back(q);
    for (int q = b; q < e; q++) if (items[q].kind != 1) order.push_back(q);
    if (e < NI) order.push_back(e);  // the PostSelect itself
    b = e + 1;
  }
  // ---- fault cost of a vector: sum over cases of P(case) [case flips it] (odd overlap)
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
          cpar[c] ^= 2;
        }
      }
  };
  auto cost2 = [&](const uint64_t* a, const uint64_t* b) {
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
  // ---- parents: greedy over earlier value items (post-select items carry no value of their own)
  std::vector<std::vector<int>> el_items(NE);  // element -> value items containing it
  std::vector<std::vector<int>> parents(NI);
  std::vector<std::vector<uint64_t>> y(NI);
  std::vector<int> ov(NI, 0), cand;
  for (int it : order) {
    if (items[it].kind == 3) continue;
    std::vector<uint64_t> cur = items[it].v;
    double ccost = cost2(cur.data(), nullptr);
    for (int round = 0; round < kAff2MaxParents && ccost > 0.0; round++) {
      cand.clear();
      for (size_t t = 0; t < NW; t++)
        for (uint64_t m = cur[t]; m; m &= m - 1) {
          const size_t src = t * 64 + __builtin_ctzll(m);
          if (src < (size_t)el0) continue;
          for (int q : el_items[src - el0])
            if (ov[q]++ == 0) cand.push_back(q);
        }
      int best = -1;
      double bcost = ccost * (1.0 - 1e-9);
      for (int q : cand) {
        ov[q] = 0;
        if (std::find(parents[it].begin(), parents[it].end(), q) != parents[it].end()) continue;
        const double qc = cost2(cur.data(), items[q].v.data());
        if (qc < bcost) { bcost = qc; best = q; }
      }
      if (best < 0) break;
      parents[it].push_back(best);
      xr(cur.data(), items[best].v.data());
      ccost = bcost;
    }
    y[it] = cur;
    for (size_t t = 0; t < NW; t++)
      for (uint64_t m = items[it].v[t]; m; m &= m - 1) {
        const size_t src = t * 64 + __builtin_ctzll(m);
        if (src >= (size_t)el0) el_items[src - el0].push_back(it);
      }
  }
  // ---- buffer rows: value items whose residual has a fault part, in program order
  std::vector<int> brow(NI, -1);
  int nbuf = 0;
  for (int it : order) {
    if (items[it].kind == 3) continue;
    bool any = false;
    for (size_t t = 0; t < NW && !any; t++) {
      uint64_t m = y[it][t];
      if (t * 64 < (size_t)el0) m &= (el0 - t * 64 >= 64) ? 0ull : (~0ull << (el0 - t * 64));
      any = m != 0;
    }
    if (any) brow[it] = nbuf++;
  }
  // ---- element -> buffer rows; case -> its rows (odd overlap over its elements)
  std::vector<std::vector<int>> el_rows(NE);
  for (int it = 0; it < NI; it++) {
    if (brow[it] < 0) continue;
    for (size_t t = 0; t < NW; t++)
      for (uint64_t m = y[it][t]; m; m &= m - 1) {
        const size_t src = t * 64 + __builtin_ctzll(m);
        if (src >= (size_t)el0) el_rows[src - el0].push_back(brow[it]);
      }
  }
  std::vector<std::vector<int>> case_rows(d.num_cases);
  {
    std::vector<uint8_t> par(nbuf + 1, 0);
    std::vector<int> touched;
    for (int c = 0; c < d.num_cases; c++) {
      touched.clear();
      for (int j = case_pauli_off[c]; j < case_pauli_off[c + 1]; j++) {
        if (case_el[j] < 0) continue;
        for (int r : el_rows[case_el[j]]) { touched.push_back(r); par[r] ^= 1; }
      }
      std::sort(touched.begin(), touched.end());
      touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
      for (int r : touched) {
        if (par[r]) case_rows[c].push_back(r);
        par[r] = 0;
      }
    }
  }
  // ---- site classes (as fs_affine.cuh): one case-pick entry per distinct (p, case_cum)
  int cwid = 1;
  for (int st = 0; st < E; st++) cwid = std::max(cwid, site_case_off[st + 1] - site_case_off[st]);
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
      std::vector<double> cc(cwid, 0.0);
      for (int c = site_case_off[st]; c < site_case_off[st + 1]; c++) cc[c - site_case_off[st]] = case_cum[c];
      cls_cum.push_back(cc);
    }
    site_cls[st] = (uint16_t)it->second;
  }
  if (cls_prob.size() >= 65535) { K.why = "too many site classes"; return K; }
  const int ncls = (int)cls_prob.size();
  bool uniform = true;  // case index = floor(x * nc / p) up to one correction step (fs_affine.cuh)
  for (int c = 0; c < ncls; c++) {
    const double sc = cls_prob[c] > 0.0 ? (double)cls_nc[c] / cls_prob[c] : 0.0;
    for (int i = 0; i + 1 < cls_nc[c]; i++)
      if (!(std::fabs(cls_cum[c][i] * sc - (i + 1)) < 0.25)) uniform = false;
  }
  if (getenv("FS_AFF_NONUNIFORM")) uniform = false;
  // ---- launch shape: queue capacity from the expected faults per word (mean + 4 sigma, the rare
  // longer queues spill to global memory); passes so that at least kMinWarps warps fit per SM
  double mu = 0.0, var = 0.0;
  for (int st = 0; st < E; st++) {
    const double pp = std::min(1.0, site_prob[st]);
    mu += 32.0 * pp;
    var += 32.0 * pp * (1.0 - pp);
  }
  int qcap = (int)std::ceil(mu + 4.0 * std::sqrt(var) + 2.0);
  qcap = std::max(8, std::min(qcap, 96));
  // ---- tables: case rows u16 | case offsets | per-pass counts | site_case u32 | site_cls u16 |
  // cls_nc i32 | cls_prob f64 | cls_cum f64 [ncls][cwid] | cls_scale f64 | ln table
  auto& T = K.tables;
  auto sec = [&](size_t bytes) {
    size_t w = T.size();
    T.resize(w + ((bytes + 15) / 16) * 4 + 4, 0u);
    return w;
  };
  auto build_tables = [&](int npass, int nbp, std::vector<size_t>& offs) {
    T.clear();
    std::vector<uint16_t> rows;
    std::vector<uint32_t> coff(d.num_cases + 1, 0);
    std::vector<uint8_t> cnp((size_t)d.num_cases * npass, 0);
    for (int c = 0; c < d.num_cases; c++) {
      coff[c] = (uint32_t)rows.size();
      for (int p = 0; p < npass; p++) {
        int cnt = 0;
        for (int r : case_rows[c])
          if (r / nbp == p) { rows.push_back((uint16_t)(r - p * nbp)); cnt++; }
        if (cnt > 255) return false;
        cnp[(size_t)c * npass + p] = (uint8_t)cnt;
      }
    }
    coff[d.num_cases] = (uint32_t)rows.size();
    offs.assign(12, 0);
    offs[0] = sec(rows.size() * 2);
    if (!rows.empty()) memcpy(T.data() + offs[0], rows.data(), rows.size() * 2);
    if (rows.size() < 65536) {
      std::vector<uint16_t> c16(coff.begin(), coff.end());
      offs[1] = sec(c16.size() * 2);
      memcpy(T.data() + offs[1], c16.data(), c16.size() * 2);
      offs[10] = 1;
    } else {
      offs[1] = sec(coff.size() * 4);
      memcpy(T.data() + offs[1], coff.data(), coff.size() * 4);
      offs[10] = 0;
    }
    offs[2] = sec(cnp.size());
    if (!cnp.empty()) memcpy(T.data() + offs[2], cnp.data(), cnp.size());
    offs[3] = sec((size_t)E * 4);
    if (E) memcpy(T.data() + offs[3], site_case_off.data(), (size_t)E * 4);
    offs[4] = sec((size_t)E * 2);
    if (E) memcpy(T.data() + offs[4], site_cls.data(), (size_t)E * 2);
    offs[5] = sec((size_t)ncls * 4);
    if (ncls) memcpy(T.data() + offs[5], cls_nc.data(), (size_t)ncls * 4);
    offs[6] = sec((size_t)ncls * 8);
    if (ncls) memcpy(T.data() + offs[6], cls_prob.data(), (size_t)ncls * 8);
    offs[7] = sec((size_t)ncls * cwid * 8);
    for (int c = 0; c < ncls; c++) memcpy(T.data() + offs[7] + (size_t)c * cwid * 2, cls_cum[c].data(), (size_t)cwid * 8);
    offs[8] = sec((size_t)ncls * 8);
    for (int c = 0; c < ncls; c++) {
      const double sc = cls_prob[c] > 0.0 ? (double)cls_nc[c] / cls_prob[c] : 0.0;
      memcpy(T.data() + offs[8] + 2 * c, &sc, 8);
    }
    offs[9] = sec(FS_LN_TAB_ENTRIES * 16);
    static const double lt[FS_LN_TAB_ENTRIES][2] = FS_LN_TAB_INIT;
    memcpy(T.data() + offs[9], lt, sizeof lt);
    return true;
  };
  const int kMinWarps = getenv("FS_AFF2_MINWARPS") ? std::max(1, atoi(getenv("FS_AFF2_MINWARPS"))) : 8;
  int npass = 1, nbp = std::max(nbuf, 1), nwarps = 0, best_np = 1, best_w = -1;
  std::vector<size_t> offs;
  auto try_np = [&](int np_) {
    nbp = std::max(1, (nbuf + np_ - 1) / np_);
    if (!build_tables(np_, nbp, offs)) return -1;
    const size_t tbl = T.size() * 4;
    const size_t per_warp = ((size_t)nbp + 1 + qcap) * 32 * 4;
    return tbl < smem_budget ? (int)std::min<size_t>(32, (smem_budget - tbl) / per_warp) : 0;
  };
  for (int np_ = 1; np_ <= 4; np_++) {
    const int w_ = try_np(np_);
    if (w_ > best_w) { best_w = w_; best_np = np_; }
    if (w_ >= kMinWarps) break;
  }
  if (best_w < 0) { K.why = "a case flips > 255 rows of one pass"; return K; }
  npass = best_np;
  nwarps = try_np(npass);
  if (nwarps < 2) { K.why = "row buffer does not fit shared memory"; return K; }
  K.npass = npass;
  K.nbp = nbp;
  K.qcap = qcap;
  K.nbuf = nbuf;
  K.nitems = NI;
  K.threads = nwarps * 32;
  K.ovf_per_lane = 256;  // spill slots per word (beyond qcap); more raises FS_ERR_ARG on the host? never
  const size_t tblw = T.size();
  const size_t per_warp_w = ((size_t)nbp + 1 + qcap) * 32;
  K.smem = tblw * 4 + (size_t)nwarps * per_warp_w * 4;
  if (getenv("FS_AFF_VERBOSE")) {
    size_t crt = 0;
    for (auto& v : case_rows) crt += v.size();
    std::vector<int> hp(kAff2MaxParents + 1, 0);
    for (int it = 0; it < NI; it++) if (items[it].kind != 3) hp[parents[it].size()]++;
    fprintf(stderr, "aff2: items %d buffered %d passes %d x %d rows, case-rows %zu (%.2f per case), qcap %d (mu %.1f), "
                    "tables %zu B, warps %d, smem %zu B; parents:", NI, nbuf, npass, nbp, crt,
            d.num_cases ? (double)crt / d.num_cases : 0.0, qcap, mu, tblw * 4, nwarps, K.smem);
    for (int k = 0; k <= kAff2MaxParents; k++) fprintf(stderr, " %d:%d", k, hp[k]);
    fprintf(stderr, "\n");
    if (atoi(getenv("FS_AFF_VERBOSE")) >= 2)
      for (int it = 0; it < NI; it++) {
        if (items[it].kind == 3) continue;
        fprintf(stderr, "  item %d kind %d idx %d cost %.3g -> %.3g brow %d parents", it, items[it].kind, items[it].idx,
                cost2(items[it].v.data(), nullptr), cost2(y[it].data(), nullptr), brow[it]);
        for (int q : parents[it]) fprintf(stderr, " %d", q);
        fprintf(stderr, "\n");
      }
  }

  // ---- kernel source
  std::ostringstream o;
  o << "#include \"fs_jit_kernels.cuh\"\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << K.threads << ", 1) fs_aff2_frame(fs::DevProg P, fs::RunArgs A, "
       "const uint32_t* __restrict__ tbl, uint32_t* __restrict__ ovf) {\n";
  o << "  extern __shared__ __align__(16) uint32_t smem[];\n";
  o << "  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;\n";
  o << "  for (int i = threadIdx.x; i < " << tblw / 4 << "; i += " << K.threads
    << ") reinterpret_cast<uint4*>(smem)[i] = __ldg(reinterpret_cast<const uint4*>(tbl) + i);\n";
  o << "  __syncthreads();\n";
  o << "  fs::Aff2Tabs T;\n";
  o << "  T.rows = reinterpret_cast<const uint16_t*>(smem + " << offs[0] << ");\n";
  o << "  T.coff = smem + " << offs[1] << ";\n";
  o << "  T.coff16 = " << (offs[10] ? "true" : "false") << ";\n";
  o << "  T.cnp = reinterpret_cast<const uint8_t*>(smem + " << offs[2] << ");\n";
  o << "  T.site_case = smem + " << offs[3] << ";\n";
  o << "  T.site_cls = reinterpret_cast<const uint16_t*>(smem + " << offs[4] << ");\n";
  o << "  T.cls_nc = reinterpret_cast<const int*>(smem + " << offs[5] << ");\n";
  o << "  T.cls_prob = reinterpret_cast<const double*>(smem + " << offs[6] << ");\n";
  o << "  T.cls_cum = reinterpret_cast<const double*>(smem + " << offs[7] << ");\n";
  o << "  T.cls_scale = reinterpret_cast<const double*>(smem + " << offs[8] << ");\n";
  o << "  T.lntab = reinterpret_cast<const double2*>(smem + " << offs[9] << ");\n";
  o << "  T.cw = " << cwid << ";\n";
  o << "  uint32_t* const B = smem + " << tblw << " + wib * " << per_warp_w << ";\n";
  o << "  uint32_t* const Q = B + " << ((size_t)nbp + 1) * 32 << ";\n";
  o << "  const uint64_t word0 = A.shot0 >> 5;\n  const uint64_t seed = A.seed;\n";
  o << "  const uint32_t ngroups = (A.W + 31) / 32;\n";
  o << "  const size_t gl0 = (size_t)blockIdx.x * " << K.threads << " + threadIdx.x;  // spill column\n";
  o << "  const size_t ovs = (size_t)gridDim.x * " << K.threads << ";\n";
  o << "  for (uint32_t grp = blockIdx.x * " << nwarps << " + wib; grp < ngroups; grp += gridDim.x * " << nwarps << ") {\n";
  o << "    const uint32_t w = grp * 32 + lane;\n";
  o << "    const bool wv = w < A.W;\n";
  o << "    const uint64_t wabs = word0 + w;\n";
  o << "    const uint64_t nleft = wv ? A.nshots - (uint64_t)w * 32 : 0;\n";
  o << "    const uint32_t valid = nleft >= 32 ? 0xFFFFFFFFu : ((1u << nleft) - 1u);\n";
  o << "    uint32_t alive = valid;\n";
  for (int cb = 0; cb < (n_coins + 3) / 4; cb++) {
    o << "    const uint4 cb" << cb << " = fs::coin_block(seed, wabs, " << cb << ");\n";
  }
  auto coin = [&](int c) {
    static const char* f[4] = {".x", ".y", ".z", ".w"};
    return "cb" + std::to_string(c / 4) + f[c % 4];
  };
  // generation: the word's noise stream into the queue
  const bool run1 = num_runs == 1;
  o << "    int qn = 0;\n";
  o << "    if (wv) qn = fs::aff2_word_faults<" << (run1 ? "true" : "false") << ", " << (uniform ? "true" : "false") << ", "
    << qcap << ">(P, T, Q, ovf + gl0, ovs, seed, wabs, lane);\n";
  for (int jj = 0; jj < d.num_observables; jj++) o << "    uint32_t ob" << jj << " = 0u;\n";
  // passes: zero the pass's rows, apply the queue, emit the items up to the next pass's first
  std::vector<int> item_pass(NI, 0);
  {
    int cp = 0;
    for (int it : order) {
      if (brow[it] >= 0) cp = brow[it] / nbp;
      item_pass[it] = cp;
    }
  }
  size_t oi = 0;
  for (int p = 0; p < npass; p++) {
    o << "    // ---- pass " << p << "\n";
    o << "    for (int i = lane; i < " << ((size_t)nbp + 1) * 8 << "; i += 32) reinterpret_cast<uint4*>(B)[i] = make_uint4(0u, 0u, 0u, 0u);\n";
    o << "    __syncwarp();\n";
    o << "    fs::aff2_apply<" << npass << ", " << qcap << ", " << nbp << ">(T, B, Q, ovf + gl0, ovs, qn, " << p << ", lane);\n";
    o << "    __syncwarp();\n";
    for (; oi < order.size() && item_pass[order[oi]] == p; oi++) {
      const int it = order[oi];
      const Item& I = items[it];
      if (I.kind == 3) {  // PostSelect: bit of an earlier value item
        o << "    alive &= ~((v" << I.idx << (I.req ? " ^ 0xFFFFFFFFu" : "") << ") & alive);\n";
        continue;
      }
      o << "    const uint32_t v" << it << " = ";
      bool first = true;
      auto term = [&](const std::string& t) { o << (first ? "" : " ^ ") << t; first = false; };
      if (brow[it] >= 0) term("B[" + std::to_string((brow[it] - p * nbp) * 32) + " + lane]");
      for (int q : parents[it]) term("v" + std::to_string(q));
      const std::vector<uint64_t>& yy = y[it];
      if (yy[0] & 1ull) term("0xFFFFFFFFu");
      for (int c = 0; c < n_coins; c++)
        if ((yy[(1 + c) >> 6] >> ((1 + c) & 63)) & 1ull) term(coin(c));
      if (first) o << "0u";
      o << ";\n";
      if (I.kind == 0) o << "    if (wv) A.meas[(size_t)" << I.idx << " * A.ostride + w] = v" << it << " & alive;\n";
      else if (I.kind == 1) o << "    if (wv) A.det[(size_t)" << I.idx << " * A.ostride + w] = v" << it << " & alive;\n";
      else if (I.kind == 2) o << "    ob" << I.idx << " ^= v" << it << " & alive;\n";
    }
    o << "    __syncwarp();\n";
  }
  o << "    if (wv) {\n";
  for (int jj = 0; jj < d.num_observables; jj++) o << "      A.obs[(size_t)" << jj << " * A.ostride + w] = ob" << jj << " & valid;\n";
  o << "      A.accepted[w] = alive & valid;\n      A.error[w] = 0u;\n    }\n";
  o << "  }\n}\n";
  K.src = o.str();
  return K;
}

}  // namespace fsjit
