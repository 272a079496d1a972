// fs_seg_check.cu -- build-time check of the headers that are otherwise only compiled at run time
// (NVRTC, per program): hand-written stand-ins for the generated segment kernels of
// fs_sampler.cu gen_segment_l / gen_segment_w, one per form (lane, lane with deferred Expands,
// warp, CTA).  `_lib.build()` compiles this to a cubin for sm_100a and discards it; nothing loads it.
#include "fs_lseg.cuh"
using namespace fs;

#define FS_CHECK_SCALARS                                                         \
  c.g_cx(1, 51, 2, 52);                                                          \
  c.g_cz(1, 51, 2, 52);                                                          \
  c.g_h(3, 53);                                                                  \
  c.g_s(4, 54);                                                                  \
  c.g_swap(5, 55, 40, 90);                                                       \
  c.meas_dstatic(3, 0, 1, 2);                                                    \
  c.meas_drandom(4, 54, 2, 0, 3, 1);                                             \
  c.noise(20);                                                                   \
  if ((c.slots >> 1) & 1u) c.xor_mask(1u, 2u, 3u, 4u);                           \
  { const uint32_t v = (0u ^ (c.slots >> 1) ^ (c.slots >> 2)) & 1u; c.detector(v, 0, 5); } \
  { const uint32_t v = (0u ^ (c.slots >> 3)) & 1u; c.obs ^= v << 0; }

#define FS_CHECK_PH(par) (par) ? make_double2(0.5, 0.1) : make_double2(0.3, 0.2), (par) ? make_double2(0.1, 0.1) : make_double2(0.9, 0.0)

extern "C" __global__ void __launch_bounds__(128) fs_check_lane(DevProg P, RunArgs A, SegArgs S, int group_bytes) {
  lseg_run<3, 0, 2, 0>(P, A, S, [&](LCtx<3, 0>& c) {
    FS_CHECK_SCALARS
    { const uint32_t par = c.fbit(4); c.expand<0>(FS_CHECK_PH(par)); }
    { const uint32_t par = c.fbit(5); c.expand<1>(FS_CHECK_PH(par)); }
    { const uint32_t par = c.fbit(6); c.expand<2>(FS_CHECK_PH(par)); }
    c.gate<FS_G_CX, 0, 2, 3>();
    c.gate<FS_G_CZ, 1, 0, 3>();
    c.gate<FS_G_H, 1, 0, 3>();
    c.gate<FS_G_S, 2, 0, 3>();
    { const uint32_t par = c.fbit(9); const double2 e0 = make_double2(0.3, 0.2), e1 = make_double2(0.3, -0.2); c.array_rot<1, 3>(par ? e1 : e0, par ? e0 : e1); }
    if (!c.measure<true, 1, 3>(5, 7, 0, 4, 3, make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0))) return;
    if (((c.slots >> 5) & 1u) != 0u) { c.alive = 0; return; }
  });
}

extern "C" __global__ void __launch_bounds__(128) fs_check_lane_local(DevProg P, RunArgs A, SegArgs S, int group_bytes) {
  lseg_run<7, 5, 6, 0>(P, A, S, [&](LCtx<7, 0>& c) {
    FS_CHECK_SCALARS
    { const uint32_t par = c.fbit(5); c.expand<5>(FS_CHECK_PH(par)); }
    { const uint32_t par = c.fbit(5); c.expand<6>(FS_CHECK_PH(par)); }
    c.gate<FS_G_CX, 0, 6, 7>();
    if (!c.measure<false, 4, 7>(5, 7, 0, 4, 3, make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0))) return;
    c.retire<4, 7>(7);
  });
}

extern "C" __global__ void __launch_bounds__(128) fs_check_lane_deferred(DevProg P, RunArgs A, SegArgs S, int group_bytes) {
  lseg_run<5, 5, 7, 2>(P, A, S, [&](LCtx<5, 2>& c) {
    FS_CHECK_SCALARS
    { const uint32_t par = c.fbit(5); c.lz0[0] = par ? make_double2(0.5, 0.1) : make_double2(0.3, 0.2); c.lz1[0] = par ? make_double2(0.1, 0.1) : make_double2(0.9, 0.0); }
    { const uint32_t par = c.fbit(6); c.lz0[1] = par ? make_double2(0.5, 0.1) : make_double2(0.3, 0.2); c.lz1[1] = par ? make_double2(0.1, 0.1) : make_double2(0.9, 0.0); }
    if (((c.slots >> 5) & 1u) != 0u) { c.alive = 0; return; }
  });
}

#define FS_CHECK_BLOCK_BODY                                                                                        \
  FS_CHECK_SCALARS                                                                                                 \
  { const uint32_t par = c.fbit(4); c.expand(256u, FS_CHECK_PH(par)); }                                            \
  c.gate(FS_G_CX, 0, 2, 512u);                                                                                     \
  c.gate(FS_G_H, 1, 0, 512u);                                                                                      \
  { const double2 ph0 = make_double2(1.0, 0.0), ph1 = ph0; c.star<false>(3, 4u, 2u, 1u, true, false, 0, ph0, ph1, 512u); } \
  { const uint32_t par = c.fbit(9); const double2 e0 = make_double2(0.3, 0.2), e1 = make_double2(0.3, -0.2); c.array_rot(1, 512u, par ? e1 : e0, par ? e0 : e1); } \
  if (!c.measure<true>(5, 7, 1, 0, 4, 3, 512u, make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0))) return; \
  if (!c.measure<false>(6, 7, 1, 0, 4, 3, 256u, make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0))) return; \
  c.retire(7, 1, 256u);                                                                                            \
  if (((c.slots >> 5) & 1u) != 0u) { c.alive = 0; return; }

extern "C" __global__ void __launch_bounds__(512, 1) fs_check_warp(DevProg P, RunArgs A, SegArgs S, int group_bytes) {
  wseg_run<32, 9>(P, A, S, group_bytes, [&](WCtxT<32>& c) { FS_CHECK_BLOCK_BODY });
}

extern "C" __global__ void __launch_bounds__(256, 3) fs_check_cta(DevProg P, RunArgs A, SegArgs S, int group_bytes) {
  wseg_run<256, 9>(P, A, S, group_bytes, [&](WCtxT<256>& c) { FS_CHECK_BLOCK_BODY });
}
