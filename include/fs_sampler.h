/*
 * fs_sampler.h -- C ABI of the B200 shot-sampling engine for the near-Clifford
 * ("Clifft"/framesim) bytecode VM.
 *
 * The reference executes a compiled BytecodeProgram one shot at a time in
 * Python (framesim/runtime.py).  This ABI replaces exactly that per-shot
 * execution layer; the compiler stays on the host.  Entry points map to the
 * reference interface as follows (paths under /root/reference/pkg/src/framesim):
 *
 *   fs_program_create   <- _compiled(prog)          runtime.py:663-669  (per-program specialisation,
 *                                                    input = BytecodeProgram backend.py:254-269)
 *   fs_sample           <- sample(prog, shots, seed, renormalize, ...)       runtime.py:777-812
 *                          run_shot(..., forced_faults, forced_outcomes)     runtime.py:731-751
 *                          (trace mode: fs_trace_in / fs_trace_out)
 *   fs_sample_host      <- the same call with host buffers (CLI `framesim sample`, cli.py:72-113)
 *   fs_accumulate       <- sample_accumulate(prog, shots, seed)              runtime.py:836-867
 *   fs_program_destroy  <- (program lifetime; Python GC in the reference)
 *   fs_last_error       <- exception text (ShotError / ValueError)           runtime.py:51-52, :785-786
 *
 * All pointers are plain C pointers.  fs_sample / fs_accumulate take DEVICE
 * pointers and a cudaStream_t passed as void*; fs_sample_host takes HOST
 * pointers and performs the host<->device copies itself.
 *
 * Output layout ("shot-bit words"): shot s of a call lives in 32-bit word
 * w = s/32, bit s%32.  W = ceil(nshots/32).
 *   meas     uint32[U][W]   user records (runtime.py:754-764 order)
 *   det      uint32[D][W]
 *   obs      uint32[O][W]
 *   accepted uint32[W]      post-selection verdict (runtime.py:632-641)
 *   error    uint32[W]      shots that raised ShotError (NaN / impossible forced outcome)
 */
#ifndef FS_SAMPLER_H
#define FS_SAMPLER_H

#ifndef __CUDACC_RTC__
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FS_ABI_VERSION 2

/* ---- serialized program (paper_2604_27058_b200/program.py) ------------------------------ */

enum fs_opcode {
  FS_OP_FRAME = 0,        /* FrameGates           backend.py:107   w1=gate_off w2=gate_cnt */
  FS_OP_ARRAY_GATE = 1,   /* ArrayGate            backend.py:114   w1=gate w2=va w3=vb w4=axa w5=axb w6=k */
  FS_OP_EXPAND = 2,       /* Expand               backend.py:126   w1=virt w2=axis w5=fp(8) w6=k_before */
  FS_OP_GAMMA_ROT = 3,    /* GammaRot             backend.py:137   w1=virt w5=fp(4) */
  FS_OP_ARRAY_ROT = 4,    /* ArrayRot             backend.py:145   w1=virt w2=axis w5=fp(4) w6=k */
  FS_OP_MEAS_DSTATIC = 5, /* MeasDormantStatic    backend.py:155   w1=virt w3=record, flip in w0 */
  FS_OP_MEAS_DRANDOM = 6, /* MeasDormantRandom    backend.py:162   w1=virt w2=coin ordinal w3=record */
  FS_OP_MEAS_ACTIVE = 7,  /* MeasActive           backend.py:169   w1=virt w2=axis w3=record w6=k */
  FS_OP_MEAS_COLLAPSE = 8,/* MeasCollapse         backend.py:189   w1..w3,w6 as above, w4=pre_off<<8|pre_cnt w5=fp(8) */
  FS_OP_RETIRE = 9,       /* Retire               backend.py:178   w1=virt w2=axis w6=k */
  FS_OP_COND_FRAME = 10,  /* CondFrame            backend.py:210   w1=pauli_off w2=pauli_cnt w3=record */
  FS_OP_NOISE = 11,       /* NoiseBlock           backend.py:219   w1=lo w2=hi w3=plan_off w4=plan_cnt */
  FS_OP_DETECTOR = 12,    /* DetectorIns          backend.py:225   w1=index w2=rec_off w3=rec_cnt */
  FS_OP_OBSERVABLE = 13,  /* ObservableIns        backend.py:231   w1=index w2=rec_off w3=rec_cnt */
  FS_OP_POSTSELECT = 14   /* PostSelectIns        backend.py:237   w1=kind(0 det,1 rec) w2=ref w3=required */
};

enum fs_gate { FS_G_H = 0, FS_G_S = 1, FS_G_SDAG = 2, FS_G_CX = 3, FS_G_CZ = 4, FS_G_SWAP = 5 };

#define FS_INS_WORDS 8
#define FS_OPCODE(w0) ((w0) & 0xFF)
#define FS_FLIP(w0) (((w0) >> 8) & 1)
#define FS_GATE_G(u) ((int)((u) >> 28))
#define FS_GATE_A(u) ((int)(((u) >> 14) & 0x3FFF))
#define FS_GATE_B(u) ((int)((u) & 0x3FFF))
#define FS_PAULI_Q(u) ((int)((u) >> 1))
#define FS_PAULI_Z(u) ((int)((u) & 1))

typedef struct fs_prog_desc {
  int32_t abi_version;       /* = FS_ABI_VERSION */
  int32_t n;                 /* qubits */
  int32_t k_max;             /* peak active dimension */
  int32_t num_instrs;
  int32_t record_count;      /* R: user + hidden records */
  int32_t num_user_records;  /* U */
  int32_t num_detectors;     /* D */
  int32_t num_observables;   /* O */
  int32_t num_sites;         /* E */
  int32_t num_slots;         /* on-chip slots for bits read after being written */
  int32_t num_fparams, num_gates, num_paulis, num_reclists, num_cases, num_plans;
  const int32_t* instrs;         /* [num_instrs][8] */
  const int32_t* schedule;       /* [num_instrs] active dimension after each instruction */
  const double* fparams;
  const uint32_t* gates;         /* g<<28 | a<<14 | b */
  const uint32_t* paulis;        /* q<<1 | is_z */
  const int32_t* reclists;
  const double* site_prob;       /* [E] */
  const int32_t* site_case_off;  /* [E+1] into case_cum */
  const double* case_cum;        /* [C] cumulative case masses (last == prob) */
  const int32_t* case_pauli_off; /* [C+1] into paulis */
  const double* cum_hazard;      /* [E+1] prefix sums of -log1p(-p) (backend.py:476-482) */
  const int32_t* plans;          /* [P][2]: (a,b) hazard segment, (-1,s) certain site */
  const int32_t* user_records;   /* [U] */
  const int32_t* record_out;     /* [R] user column or -1 */
  const int32_t* bit_slot;       /* [R+D] slot of record/detector bit or -1 */
} fs_prog_desc;

/* ---- sampling flags ------------------------------------------------------------------------ */
#define FS_RNG_PHILOX   0u   /* default: Philox4x32-10 keyed by (seed, shot|word, instruction) */
#define FS_RNG_SPLITMIX 1u   /* reference stream: framesim ShotRng draw for draw (rng.py:24-71) */
#define FS_NO_RENORM    2u   /* renormalize=False (runtime.py:355-366, :389-404) */
#define FS_FORCE_GENERAL 4u  /* testing: force the general per-shot-lane interpreter */
#define FS_FORCE_HBM    8u   /* testing: force the large-k (HBM-resident array) engine */
#define FS_NO_JIT       16u  /* testing: frame engine interpreter instead of the program-specialised kernel */
#define FS_FORCE_SEGMENTED 32u /* testing: post-selected programs run segment by segment (survivor
                                  compaction, warp/CTA-per-shot block engine) also in trace mode */

/* trace mode: every random choice may be supplied (SURVEY §8(d) "trace mode"), and the state can
 * be read back at the end and at a list of checkpoints in ONE call (run_shot(..., trace=)
 * runtime.py:731-751 calls its callback after every instruction, :745-748). */
typedef struct fs_trace_in {
  const int16_t* fault_modes; /* [nshots][E] runtime.py:587-601 encoding: 0 sample, 1 trigger with
                                 random case, 2 off, 3+c case c.  NULL = free hazard sampling. */
  const int8_t* forced;       /* [nshots][R]: -1 free, 0/1 forced outcome.  NULL = all free. */
  int32_t stop;               /* execute instructions [0, stop); <0 = whole program */
  int32_t ncheckpoints;       /* number of checkpoints (0 = none) */
  const int32_t* checkpoints; /* HOST memory, [ncheckpoints] strictly ascending instruction counts
                                 in [0, stop]: checkpoint c = the state after instructions [0, c),
                                 i.e. what the reference trace callback sees after instrs[c-1] */
} fs_trace_in;

typedef struct fs_trace_out {  /* any member may be NULL */
  uint8_t* frame_x;   /* [nshots][n] */
  uint8_t* frame_z;   /* [nshots][n] */
  double* gamma;      /* [nshots][2] */
  double* amps;       /* [nshots][2^k_stop][2] active array at the stop point */
  uint32_t* draws;    /* [nshots] random draws consumed (FS_RNG_SPLITMIX) */
  uint8_t* records;   /* [nshots][R] every record bit, user and hidden (ShotState.records) */
  /* per checkpoint j (fs_trace_in.checkpoints[j]); a shot that halted (PostSelect) or raised
     before the checkpoint has cp_valid 0 and unspecified state there */
  uint8_t* cp_valid;    /* [ncp][nshots] */
  uint8_t* cp_frame_x;  /* [ncp][nshots][n] */
  uint8_t* cp_frame_z;  /* [ncp][nshots][n] */
  double* cp_gamma;     /* [ncp][nshots][2] */
  double* cp_amps;      /* checkpoint blocks back to back: block j = [nshots][2^k_j][2] with
                           k_j = schedule[checkpoints[j] - 1] (0 when checkpoints[j] == 0) */
} fs_trace_out;

typedef struct fs_sample_out {
  uint32_t* meas;      /* [U][W] */
  uint32_t* det;       /* [D][W] */
  uint32_t* obs;       /* [O][W] */
  uint32_t* accepted;  /* [W] */
  uint32_t* error;     /* [W] */
  int32_t* status;     /* optional [1]: max FS_ERR_SHOT_* raised (same memory space as the rest) */
} fs_sample_out;

/* status codes */
#define FS_OK 0
#define FS_ERR_ARG -1
#define FS_ERR_CUDA -2
#define FS_ERR_SHOT_NAN 1        /* "NaN amplitude encountered at an active measurement" */
#define FS_ERR_SHOT_FORCED 2     /* "forced outcome ... has probability ..." */

#ifndef __CUDACC_RTC__ /* host entry points (not visible to NVRTC-compiled device code) */
int fs_abi_version(void);
const char* fs_last_error(void);

typedef struct fs_prog fs_prog;

/* Copies the program to the current CUDA device; chooses the execution engine. */
int fs_program_create(const fs_prog_desc* desc, fs_prog** out);
void fs_program_destroy(fs_prog* prog);
/* engine chosen for a flag set: 0 = general (lane = shot), 1 = bit-sliced frame engine,
   2 = large-k engine (active arrays in HBM) */
int fs_program_engine(const fs_prog* prog, uint32_t flags);

/* shot0 must be a multiple of 32: the Philox stream keys coins and noise by the absolute 32-shot
 * word (shot / 32) and Born draws by the absolute shot, so any split of a run into calls at
 * multiples of 32 reproduces it exactly (FS_RNG_SPLITMIX is keyed per shot, like framesim).
 * Returns FS_OK, or FS_ERR_SHOT_* when some shot raised (see out->error), or a negative error. */
int fs_sample(fs_prog* prog, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
              const fs_trace_in* tin, const fs_sample_out* out, const fs_trace_out* tout,
              void* stream);
int fs_sample_host(fs_prog* prog, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                   const fs_trace_in* tin, const fs_sample_out* out, const fs_trace_out* tout);

/* counts (device int64): [U] meas, [D] det, [O] obs, then accepted; sums over ACCEPTED shots
 * (runtime.py:857-865).  Returns FS_OK, or FS_ERR_SHOT_* when some shot raised ShotError (the
 * reference's sample_accumulate propagates it); reading that status synchronizes the stream. */
int fs_accumulate(fs_prog* prog, uint64_t seed, uint64_t shot0, uint64_t nshots, uint32_t flags,
                  int64_t* counts, void* stream);

/* The reference CLI's sample formats (cli.py:66-69, :94-109), produced on the device from the
 * shot-bit words of an fs_sample call over `nshots` shots (row stride ceil(nshots/32)).  Record
 * bits = user measurements ++ detectors ++ observables; a shot is written when accepted or
 * keep_rejected.  FS_FMT_01: '0'/'1' chars + " rejected" (keep_rejected, not accepted) + '\n';
 * FS_FMT_BIN: np.packbits(bits, bitorder="little"); FS_FMT_CSV: "<index>,<weight_text>,<bits>\n"
 * with index = index0 + position among the written records (the header line is the caller's).
 * dst: device buffer of `cap` bytes (>= fs_format_bound).  *nbytes / *nkept (host) = bytes and
 * records written. */
#define FS_FMT_01 0
#define FS_FMT_BIN 1
#define FS_FMT_CSV 2
int fs_format(fs_prog* prog, const fs_sample_out* words, uint64_t nshots, int format, int keep_rejected,
              uint64_t index0, const char* weight_text, uint8_t* dst, uint64_t cap, uint64_t* nbytes,
              uint64_t* nkept, void* stream);
uint64_t fs_format_bound(const fs_prog* prog, uint64_t nshots, int format, uint64_t index0,
                         const char* weight_text);

/* Stratified importance sampling (runtime.py:886-945): every shot conditioned on exactly w
 * realised faults.  fs_stratum_weight = StratumSpec(prog, w).weight = Pr[W = w] (FS_ERR_ARG with
 * "stratum fault count w exceeds E sites" when w > E).  The forced sites of a shot are drawn by
 * StratumSpec.draw_forced's sequential conditioning: FS_RNG_SPLITMIX consumes the shot's reference
 * stream exactly like the reference (records identical to framesim.sample(..., stratum=)); the
 * Philox stream uses its own draws.  Outputs / accumulate as fs_sample / fs_accumulate. */
int fs_stratum_weight(fs_prog* prog, uint32_t w, double* weight);
int fs_sample_stratum(fs_prog* prog, uint32_t w, uint64_t seed, uint64_t shot0, uint64_t nshots,
                      uint32_t flags, const fs_sample_out* out, void* stream);
int fs_sample_stratum_host(fs_prog* prog, uint32_t w, uint64_t seed, uint64_t shot0, uint64_t nshots,
                           uint32_t flags, const fs_sample_out* out);
int fs_accumulate_stratum(fs_prog* prog, uint32_t w, uint64_t seed, uint64_t shot0, uint64_t nshots,
                          uint32_t flags, int64_t* counts, void* stream);

/* expectation_probe traversal (runtime.py:951-989): for the device active array amps[2^k][2],
 * out[0] = Re sum_idx conj(a[idx ^ xm]) i^ycount (-1)^popcount(idx & zm) a[idx],
 * out[1] = sum |a|^2 (host doubles).  The Pauli mapping through the final tableau, the frame
 * parity and the sign stay with the caller (host compiler objects). */
int fs_probe(const double* amps, int32_t k, uint64_t xm, uint64_t zm, int32_t ycount, double* out, void* stream);
#endif

#ifdef __cplusplus
}
#endif
#endif
