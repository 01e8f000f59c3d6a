/* vscreen_gpu C-ABI — the drop-in boundary of the B200 dock-and-score path.
 *
 * Plain C: POD structs, raw pointers and sizes, int status codes, no
 * exceptions and no torch types.  One handle per host thread / GPU; handles
 * are not shared between threads.  All host buffers are caller-owned.
 *
 * The reference has no FFI layer for this path: its boundary is the C++
 * header API (proj/include/vscreen/{dock,batcher,chem,pipeline}.hpp) plus
 * the pybind11 module (proj/bindings/module.cpp).  Each entry point below
 * names the reference function it replaces; include/vscreen_gpu/vscreen_gpu.hpp
 * maps these status codes back onto the reference exception types so C++
 * callers compile unchanged, and paper_2304_09953_b200/ is the Python mirror.
 */
#ifndef VSCREEN_GPU_CAPI_H
#define VSCREEN_GPU_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------- status -- */
enum vs_status {
  VS_OK = 0,
  VS_ERR_INVALID_ARGUMENT = -1, /* std::invalid_argument   dock.cpp:322-323 */
  VS_ERR_ATOM_COUNT = -2,       /* dock::AtomCountMismatch dock.cpp:219-230,299-301,324 */
  VS_ERR_EMPTY_BOUNDS = -3,     /* dock::EmptyBounds       dock.cpp:321 */
  VS_ERR_LENGTH = -4,           /* dock::LengthMismatch    dock.cpp:393-396 */
  VS_ERR_OUT_OF_RANGE = -5,     /* batcher::OutOfRange     batcher.cpp:23-25,161 */
  VS_ERR_ITEM_TOO_LARGE = -6,   /* batcher::ItemTooLarge   batcher.cpp:31-34 */
  VS_ERR_POCKET = -7,           /* std::runtime_error      dock.cpp:441,448 */
  VS_ERR_PARSE = -8,            /* chem::ParseError        chem.cpp:109-264 */
  VS_ERR_CAPACITY = -9,         /* ligand beyond GPU limits (atoms>128, torsions>64,
                                   restarts>64, flex_angles>16) or buffer too small */
  VS_ERR_CUDA = -10,
  VS_ERR_NO_DEVICE = -11,
  VS_ERR_STATE = -12,           /* call order (e.g. dock before pocket/library) */
  VS_ERR_DISCONNECTED = -13,    /* chem::DisconnectedGraph chem.cpp:408 */
  VS_ERR_FORMAT = -14           /* codec::BadFormat / UnknownCode codec.cpp:147-161, 195-289 */
};

/* ------------------------------------------------------------- pocket -- */
/* dock::Site (dock.hpp:18-23); kind 0 steric, 1 hbond, 2 lipophilic */
typedef struct {
  double center[3];
  double weight;
  double sigma;
  int32_t kind;
  int32_t reserved;
} vs_site;

/* dock::Pocket (dock.hpp:32-37) */
typedef struct {
  const vs_site* sites;
  int32_t n_sites;
  int32_t reserved;
  double lo[3];
  double hi[3];
  double clash_radius;
  double clash_penalty;
} vs_pocket;

/* ------------------------------------------------------------ library -- */
/* A ligand library in the reference's own types, flattened: chem::Conformer
 * coords (chem.hpp:78-81, FP64), dock::TorsionTopology axes and moving lists
 * (dock.hpp:65-71), the element class used by rescore (dock.cpp:309), the
 * per-ligand dock seed (pipeline.cpp:483) and the rank of the ligand id in
 * std::map order (the rank_ligands tie-break, pipeline.cpp:243-251). */
typedef struct {
  int32_t n_ligands;
  int32_t reserved;
  const int32_t* n_atoms;      /* [n] */
  const int32_t* n_tors;       /* [n] */
  const int32_t* rot_bonds;    /* [n] descriptor for size classes (may be NULL: = n_tors) */
  const double* coords;        /* [sum n_atoms][3] */
  const int32_t* atom_class;   /* [sum n_atoms] 0 other, 1 C, 2 N or O */
  const int32_t* axis_a;       /* [sum n_tors] */
  const int32_t* axis_b;       /* [sum n_tors] */
  const int32_t* moving_count; /* [sum n_tors] */
  const int32_t* moving;       /* [sum moving_count] */
  const uint64_t* seeds;       /* [n] */
  const uint32_t* id_rank;     /* [n] */
} vs_library;

/* batcher::SizeClass (batcher.hpp:33-40), half-open ranges */
typedef struct {
  int32_t atom_lo, atom_hi, rot_lo, rot_hi;
} vs_size_class;

/* ------------------------------------------------------------- params -- */
/* dock(restarts, diversity_delta, seed, max_steps) (dock.hpp:107-109) plus
 * StageKnobs keep_top/min_score (pipeline.hpp:33-40) and the sweep-v1
 * knobs (docs/SWEEP_V1.md).  max_steps of the reference ascent has no
 * meaning for sweep-v1 and is not taken. */
typedef struct {
  int32_t restarts;        /* R >= 1, <= 64 */
  int32_t rotations;       /* K >= 1 */
  int32_t flex_angles;     /* A in [1, 16] */
  int32_t flex_passes;     /* F >= 0 */
  double diversity_delta;  /* >= 0 */
  int32_t keep_top;        /* >= 0 */
  int32_t write_all_poses; /* also return every kept pose (dock() output) */
  double min_score;
  uint64_t rotation_seed;
  int32_t polish;          /* 0 off, 1 rigid compass, 2 + fine torsion pass (SWEEP_V1.md §3.5) */
  int32_t reserved;
} vs_dock_params;

/* One pose (dock::Pose, dock.hpp:39-46) in FP32 plus its sweep-v1 index
 * tuple.  Torsions are returned in a parallel array. */
typedef struct {
  float t[3];
  float q[4]; /* w, x, y, z */
  float score;
  float rescore;
  int16_t restart;
  int16_t attempt;
  int16_t rot;
  int16_t reserved;
} vs_pose;

/* Results of one dock run, caller-owned host buffers.  Ligand i's torsion
 * block starts at tors_off(i) * slots where tors_off is the prefix sum of
 * n_tors and slots = keep_top (surv) or restarts (all). */
typedef struct {
  float* best;        /* [n] max rescore over survivors; -inf when dropped */
  int32_t* n_kept;    /* [n] kept (diverse) poses; -1 = out of every size class */
  int32_t* n_surv;    /* [n] poses surviving filter_poses */
  vs_pose* surv;      /* [n * keep_top] */
  float* surv_tors;   /* [sum n_tors * keep_top] */
  vs_pose* all;       /* optional [n * restarts] */
  float* all_tors;    /* optional [sum n_tors * restarts] */
  uint64_t* keys;     /* optional [n] top-k keys */
} vs_results;

typedef struct vs_handle vs_handle;

/* Page-locked host memory (cudaHostAlloc, portable): library arrays and
 * result buffers placed here move at full link rate, and vs_fetch_results /
 * vs_dock_host DMA straight into result buffers that live in it. */
int vs_host_alloc(int64_t bytes, void** out);
int vs_host_free(void* p);

/* ------------------------------------------------------ GPU runtime ----- */
int vs_create(int device, vs_handle** out);
void vs_destroy(vs_handle* h);
const char* vs_last_error(const vs_handle* h);
/* name (<= 255 chars), SM count, SM clock (kHz) */
int vs_device_info(const vs_handle* h, char* name, int32_t* sm_count, int32_t* clock_khz);

/* Upload the pocket (parse_pocket_json result, dock.cpp:432) and, when
 * grid_spacing > 0, build the three FP32 grid maps (steric / hbond /
 * lipophilic) over bounds +- grid_pad on the device.  Validation as
 * dock.cpp:321, 441, 448. */
int vs_set_pocket(vs_handle* h, const vs_pocket* pocket, double grid_spacing, double grid_pad);
int vs_grid_info(const vs_handle* h, int32_t dims[3], float origin[3], float* spacing);
int vs_grid_fetch(vs_handle* h, float* steric, float* hbond, float* lipo);

/* Pack the library into the device SoA (size-class buckets, LPT order
 * within a bucket) and upload it.  classes == NULL: automatic atom-count
 * buckets.  Ligands outside every class are dropped (pipeline.cpp:447-452). */
int vs_upload_library(vs_handle* h, const vs_library* lib, const vs_size_class* classes,
                      int32_t n_classes);
/* Run the path on the resident library; stream = cudaStream_t or NULL. */
int vs_dock(vs_handle* h, const vs_dock_params* params, void* stream);
int vs_fetch_results(vs_handle* h, vs_results* out);
/* Upload + dock + fetch in one call (host buffers in and out). */
int vs_dock_host(vs_handle* h, const vs_library* lib, const vs_size_class* classes,
                 int32_t n_classes, const vs_dock_params* params, vs_results* out);
/* vs_dock_host for L, and the device pack of `next` (may be NULL) started on
 * the handle's copy stream so that its transfer and packer kernels run under
 * this dock: the next call with next's library (same arrays, same classes)
 * adopts it without a transfer.  A stream of libraries then moves each one to
 * the device while the previous one docks.  The caller keeps next's arrays
 * alive and unchanged until that call.  A `next` the packer rejects is not
 * prefetched; the call that docks it reports the error. */
int vs_dock_host_prefetch(vs_handle* h, const vs_library* L, const vs_library* next,
                          const vs_size_class* classes, int32_t nc, const vs_dock_params* prm,
                          vs_results* out);
/* Device time (ms, CUDA events on the launch stream) of the dock kernels of
 * the last vs_dock call, and the number of kernels this handle launched. */
double vs_last_dock_ms(const vs_handle* h);
uint64_t vs_launch_count(const vs_handle* h);
/* Device time (ms) of the last vs_dock split by kernel: [0] start, [1] sweep,
 * [2] flex+keep, [3] finish (staged mode; the fused kernel reports its whole
 * time in [2]).  CUDA events around every launch on the launch stream. */
int vs_last_phase_ms(vs_handle* h, double out[4]);
/* the same split with the polish kernel on its own, up to n entries (returns
 * how many were written): [0] start, [1] sweep, [2] flex+keep, [3] finish,
 * [4] polish (vs_last_phase_ms counts [4] in [2]) */
int vs_last_phase_ms_ex(vs_handle* h, double* out, int32_t n);
/* work counters of the last vs_dock: [0] translation-sweep iterations,
 * [1] the same weighted by ligand atoms, [2] start attempts, [3] flex pair
 * softplus evaluations (pairs inside the cutoff), [4..7] SM cycles summed
 * over warps in the start, sweep, flex and keep phases */
int vs_last_stats(vs_handle* h, uint64_t out[8]);
/* the same, up to n counters (returns how many were written): [8] rigid
 * compass iterations after the flex (polish), [9] the same weighted by
 * ligand atoms ([0]/[1] then count the sweep's lattice or compass only) */
int vs_last_stats_ex(vs_handle* h, uint64_t* out, int32_t n);
/* measured device peaks (ops/s): FP32 FMA (2 flops), FP64 FMA, MUFU ex2 */
int vs_measure_peaks(vs_handle* h, double* fp32_flops, double* fp64_flops, double* xu_ops);
/* measured random-gather peak (16 B loads/s): independent ld.global.nc.v4 of
 * uniformly random cells of an L2-resident 8 MB array, every lane a distinct
 * sector, full occupancy and 8 loads in flight per thread -- the access
 * pattern of the sweep key lookups at the most memory-level parallelism */
int vs_measure_gather_peak(vs_handle* h, double* loads_per_s);
/* the same with 16 B (FP16 key cell) or 32 B (ld.global.nc.v8.f32, one FP32
 * corner cell = one sector: the L2-gather roof of SURVEY §8(d), whose L2_B
 * counts 8 corners x 4 B per lookup) loads; 16 MB array for 32 B */
int vs_measure_gather_peak_ex(vs_handle* h, int32_t bytes_per_load, double* loads_per_s);

/* Global top-k of the last run: keys ascending = (score desc, id_rank asc)
 * (rank_ligands, pipeline.cpp:243-251).  key = (~orderable(score) << 32) |
 * id_rank; dropped ligands are ~0. */
int vs_topk(vs_handle* h, int32_t k, uint64_t* out_keys);
int vs_topk_device(vs_handle* h, int32_t k, uint64_t* out_keys_dev, void* stream);
/* Merge of gathered per-rank top-k keys (device buffers). */
int vs_topk_merge_device(vs_handle* h, const uint64_t* keys_dev, int64_t n, int32_t k,
                         uint64_t* out_keys_dev, void* stream);

/* Multi-GPU (the reference has no collective: its callers
 * run dock() on std::threads, pipeline.cpp:29-55, 482-486).  One process or
 * thread per GPU, a contiguous shard of the library each; the only exchange
 * is the top-k: vs_topk_allgather = local top-k -> one ncclAllGather of k
 * u64 keys per rank -> the same device merge on every rank, all on `stream`.
 * The communicator is either created here (rank 0 calls vs_nccl_unique_id
 * and the caller broadcasts the 128 bytes, NCCL's usual bootstrap) or an
 * existing ncclComm_t is attached / passed per call.  libnccl.so.2 is
 * resolved at run time (the copy already loaded in the process, else the
 * system's); VS_ERR_NO_DEVICE when there is none. */
#define VS_NCCL_ID_BYTES 128
int vs_nccl_unique_id(uint8_t out[VS_NCCL_ID_BYTES]);
int vs_comm_init(vs_handle* h, int32_t nranks, int32_t rank, const uint8_t id[VS_NCCL_ID_BYTES]);
int vs_comm_attach(vs_handle* h, void* nccl_comm /* ncclComm_t, not owned */);
void vs_comm_destroy(vs_handle* h);
/* comm = ncclComm_t or NULL (the handle's own); out_keys_dev: k device keys */
int vs_topk_allgather(vs_handle* h, void* nccl_comm, int32_t k, uint64_t* out_keys_dev,
                      void* stream);
float vs_key_score(uint64_t key);
uint32_t vs_key_id_rank(uint64_t key);

/* score_gradient (dock.cpp:284-295, Objective::grad :117-160) of given
 * poses, FP64 on the GPU (analytic pocket; the grid is not used): score,
 * d/dt (3 per pose), tangent-projected d/dq (4 per pose, w x y z) and
 * central-difference d/dtorsion (h = 1e-5; n_tors of the pose's ligand per
 * pose, in pose order).  Poses are FP64 (reference Pose). */
int vs_score_gradient(vs_handle* h, const vs_library* lib, int64_t n_poses,
                      const int32_t* pose_lig, const double* t, const double* q,
                      const double* tors, double* score, double* grad_t, double* grad_q,
                      double* grad_tors);
/* geometric_score + rescore of given poses (dock.cpp:278, 297).  pose_lig
 * must be non-decreasing; torsions of pose p are tors[tors_off_p ...] in
 * pose order, n_tors of its ligand each. */
int vs_rescore(vs_handle* h, const vs_library* lib, int64_t n_poses, const int32_t* pose_lig,
               const float* t, const float* q, const float* tors, float* geo, float* resc);
/* the same with the length of `tors` checked against the poses' ligands
 * (AtomCountMismatch, check_counts dock.cpp:219-230); n_tors_values < 0
 * skips the check (= vs_rescore) */
int vs_rescore_checked(vs_handle* h, const vs_library* lib, int64_t n_poses,
                       const int32_t* pose_lig, const float* t, const float* q, const float* tors,
                       int64_t n_tors_values, float* geo, float* resc);
/* The reference ascent (dock.cpp:168-203: Armijo, step 0.5, shrink 0.5,
 * c 1e-4, |g| < 1e-6) from the given poses, one warp per pose on the
 * device, FP64 score_gradient arithmetic; t[3n], q[4n] (w, x, y, z) and the
 * concatenated torsions are updated in place; score[n] and steps[n]
 * (accepted steps) optional.  Quality-only refinement. */
int vs_ascend(vs_handle* h, const vs_library* lib, int64_t n_poses, const int32_t* pose_lig,
              double* t, double* q, double* tors, int32_t max_steps, double* score,
              int32_t* steps);
/* The same rescoring for poses already in device memory, against the
 * resident library (vs_upload_library): pose_lig / t / q / tors / geo /
 * resc are device pointers (layout as vs_rescore), all work on `stream`. */
int vs_rescore_device(vs_handle* h, int64_t n_poses, const int32_t* pose_lig, const float* t,
                      const float* q, const float* tors, float* geo, float* resc, void* stream);
/* The survivors of the last vs_dock (still in device memory) re-scored
 * against the current pocket, e.g. finer maps set by vs_set_pocket after
 * the dock (BASELINE config 5): geo / resc device arrays [n * keep_top],
 * slot l * keep_top + k for k < n_surv[l] (other slots untouched). */
int vs_rescore_survivors(vs_handle* h, float* geo, float* resc, void* stream);

/* geometric_score / rescore (dock.cpp:278-282, 297-316) of given poses in
 * FP64 on the device (the score_gradient arithmetic without the gradient;
 * analytic pocket): geo[n], resc[n] optional.  The drop-in's per-pose
 * scoring (include/vscreen/dock.hpp). */
int vs_score64(vs_handle* h, const vs_library* lib, int64_t n_poses, const int32_t* pose_lig,
               const double* t, const double* q, const double* tors, double* geo, double* resc);

/* Refined dock results (caller-owned): ligand i's poses at slots
 * i * restarts + r, r < n_poses[i], sorted by score descending; torsions at
 * tors_off(i) * restarts + r * n_tors(i).  q is unit (pose_of, dock.cpp:210). */
typedef struct {
  int32_t* n_poses; /* [n]; -1 = out of every size class */
  double* t;        /* [n * restarts * 3] */
  double* q;        /* [n * restarts * 4] (w, x, y, z) */
  double* tors;     /* [sum n_tors * restarts] */
  double* score;    /* [n * restarts] FP64 geometric score of the refined pose */
  int32_t* restart; /* [n * restarts] optional: the restart each pose came from */
} vs_refined;
/* dock() with the reference's contract (dock.cpp:318-371): the sweep-v1
 * restarts (vs_dock, every kept pose) each refined by the reference ascent
 * (vs_ascend, max_steps), then the reference's keep rule on the refined
 * coordinates in restart order (RMSD >= diversity_delta from every kept
 * pose) and a stable sort by score descending. */
int vs_dock_refined_host(vs_handle* h, const vs_library* lib, const vs_size_class* classes,
                         int32_t n_classes, const vs_dock_params* params, int32_t max_steps,
                         vs_refined* out);

/* Device time (ms, CUDA events on the launch stream) of the rescore kernels
 * of the last vs_rescore call (-1 before the first). */
double vs_last_rescore_ms(const vs_handle* h);
/* The restart start draws of the device dock (dock.cpp:343-354, Rng
 * rng.hpp:14-41) for every (ligand, restart r < restarts, attempt a <
 * attempts): row ((i * restarts) + r) * attempts + a of `out` (stride
 * floats) holds t[3], q[4] (w, x, y, z) and theta[n_tors[i]] as the FP32
 * values the dock starts from.  Needs a pocket (the box bounds t is drawn
 * in).  Parity instrument: the same device code as the start kernel. */
int vs_start_draws(vs_handle* h, const uint64_t* seeds, const int32_t* n_tors, int32_t n,
                   int32_t restarts, int32_t attempts, int32_t stride, float* out);

/* --------------------------------------------------- host-side (CPU) --- */
/* Rng(seed).split(path...) then n next_u64 (rng.hpp:14-21) */
int vs_rng_u64(uint64_t seed, const uint64_t* path, int32_t depth, int32_t n, uint64_t* out);
/* corpus::random_smiles(Rng(seed).split(i)) (tools/smiles_corpus.hpp:13) */
int vs_random_smiles(uint64_t seed, uint64_t i, char* out, int32_t cap);

/* One ligand: parse_smiles + rotatable_bonds + embed_3d + torsion_topology
 * (chem.cpp:109,319,406; dock.cpp:234).  iterations < 0: no embedding. */
typedef struct {
  int32_t cap_atoms, cap_bonds, cap_tors, cap_moving;
  int32_t n_atoms, n_bonds, n_tors, n_moving, rot_bonds;
  int32_t parse_kind, parse_pos; /* on VS_ERR_PARSE */
  double* coords;                /* [cap_atoms*3] */
  int32_t* atom_class;           /* [cap_atoms] */
  char* elements;                /* [cap_atoms*3] NUL-padded element symbols */
  uint8_t* aromatic;             /* [cap_atoms] */
  int32_t* bonds;                /* [cap_bonds*3] a, b, order */
  uint8_t* ring;                 /* [cap_bonds] */
  int32_t* axis_a;               /* [cap_tors] */
  int32_t* axis_b;
  int32_t* moving_count;
  int32_t* moving;               /* [cap_moving] */
} vs_ligand_buf;
int vs_ligand_build(const char* smiles, uint64_t embed_seed, int32_t iterations,
                    vs_ligand_buf* out);

/* Many ligands on `threads` host threads.  smiles: NUL-separated blob.
 * iterations >= 0: embed_3d on the host with that many spring iterations;
 * -1: zero coordinates; VS_EMBED_PLACE_ONLY: the BFS placement only, to be
 * relaxed on the device by vs_libbuild_relax (GPU embed_3d). */
#define VS_EMBED_PLACE_ONLY (-2)
/* parse + topology only; embed_3d entirely on the device by vs_libbuild_embed */
#define VS_EMBED_DEVICE (-3)
typedef struct vs_libbuild vs_libbuild;
int vs_libbuild_run(const char* smiles_blob, int32_t n, const uint64_t* embed_seeds,
                    int32_t iterations, int32_t threads, vs_libbuild** out);
/* totals and per-ligand status (0 ok, VS_ERR_PARSE, VS_ERR_DISCONNECTED) */
int vs_libbuild_sizes(const vs_libbuild* b, int64_t* atoms, int64_t* tors, int64_t* moving);
int vs_libbuild_fetch(const vs_libbuild* b, int32_t* status, int32_t* n_atoms, int32_t* n_tors,
                      int32_t* rot_bonds, double* coords, int32_t* atom_class, int32_t* axis_a,
                      int32_t* axis_b, int32_t* moving_count, int32_t* moving);
void vs_libbuild_free(vs_libbuild* b);
/* The spring relaxation of embed_3d (chem.cpp:355-392, 434-445: `iterations`
 * steps, then up to 20 rounds of 50 while the closest pair is < 0.5 A) on the
 * device for every ligand built with VS_EMBED_PLACE_ONLY; FP64 in the
 * reference's operation order, bit-identical to the host embed. */
int vs_libbuild_relax(vs_handle* h, vs_libbuild* b, int32_t iterations);
/* The whole embed_3d (chem.cpp:404-446) on the device for every ligand built
 * with VS_EMBED_DEVICE: the BFS tetrahedral placement with the reference Rng
 * jitter (Box-Muller in CUDA FP64 log / cos, which may differ from glibc in
 * the last bit, so the coordinates match the host embed to a tolerance, not
 * bit for bit), then the relaxation above. */
int vs_libbuild_embed(vs_handle* h, vs_libbuild* b, int32_t iterations);
/* synthetic libraries from the reference corpus sampler: indices i of the
 * first n_want entries random_smiles(Rng(seed).split(i)) within the atom /
 * torsion bounds (inclusive); then build those entries */
int vs_corpus_select(uint64_t seed, int64_t n_want, int32_t atom_lo, int32_t atom_hi,
                     int32_t tors_lo, int32_t tors_hi, int64_t max_scan, int32_t threads,
                     int64_t* out_index);
int vs_libbuild_corpus(uint64_t seed, const int64_t* index, int32_t n, const uint64_t* embed_seeds,
                       int32_t iterations, int32_t threads, vs_libbuild** out);
/* flexible ligands (C4): consecutive corpus entries concatenated until
 * >= atom_lo atoms; accepted ligand k is entries [first[k], first[k]+count[k]).
 * The index space is scanned in fixed chunks of 16384 entries (each chunk
 * from its own first entry) on all host threads; the selection does not
 * depend on the thread count. */
int vs_flexible_select(uint64_t seed, int32_t n_want, int32_t atom_lo, int32_t atom_hi,
                       int32_t tors_lo, int32_t tors_hi, int64_t max_scan, int64_t* first,
                       int32_t* count);

/* SMZC library decompression (codec.cpp:147-161, 195-289; ingest row f2):
 * dict = the SMZ1 dictionary file bytes, data = the .smzc file bytes; out
 * receives the reference's decompress_stream text (every record + '\n'),
 * expanded on `threads` host threads.  out = NULL: size query (*out_len).
 * VS_ERR_FORMAT on a bad magic, a dictionary hash mismatch (SHA-256),
 * truncation or an unknown code byte (vs_codec_last_error has the text). */
int vs_smzc_decompress(const uint8_t* dict, int64_t dict_len, const uint8_t* data, int64_t len,
                       int32_t threads, char* out, int64_t cap, int64_t* out_len);
const char* vs_codec_last_error(void);
/* codec::load_dictionary (codec.cpp:188-215): validate an SMZ1 dictionary;
 * *n_entries = its entry count.  VS_ERR_FORMAT with the reference's message. */
int vs_smz1_check(const uint8_t* dict, int64_t dict_len, int32_t* n_entries);
/* SHA-256 (FIPS 180-4) of len bytes: codec::dictionary_sha256 over the SMZ1
 * bytes of a dictionary (codec.cpp:222-229) */
int vs_sha256(const uint8_t* data, int64_t len, uint8_t* out32);

/* JSON number text (dock.cpp:460-489, pipeline.cpp:269-301): x[i] as the
 * reference's nlohmann::json dump prints it, NUL-terminated at out + i*stride.
 * VS_ERR_CAPACITY if a text needs stride bytes or more. */
int vs_json_format_doubles(const double* x, int64_t n, char* out, int32_t stride);

/* batcher (batcher.cpp:7-86) */
int vs_default_classes(vs_size_class* out, int32_t cap);
int vs_size_class_of(int32_t atoms, int32_t rot, const vs_size_class* classes, int32_t n);
int vs_target_batch_size(const vs_size_class* cls, double memory_capacity, double mem_fixed,
                         double mem_per_atom, double mem_per_rotbond, int64_t* out);
double vs_simulate_throughput(int64_t n_items, double launch_overhead, double service_time);
/* dock-stage bucket replay of run_campaign (pipeline.cpp:439-461): per
 * ligand in_range[i]; batches as (class, length) + flattened members.
 * Returns the number of batches (or a negative status). */
int vs_bucket_replay(const int32_t* atoms, const int32_t* rot, int32_t n,
                     const vs_size_class* classes, int32_t n_classes, double memory_capacity,
                     double mem_fixed, double mem_per_atom, double mem_per_rotbond,
                     double max_age, int32_t* in_range, int32_t* batch_cls, int32_t* batch_len,
                     int32_t* batch_members);
/* dock seeds Rng(master).split(2).split(i), i = post-compaction index
 * (pipeline.cpp:481-484) */
int vs_campaign_seeds(uint64_t master_seed, int32_t stage, const int32_t* in_range, int32_t n,
                      uint64_t* out);
/* host merge of top-k keys (e.g. gathered per-rank top-k on a CPU caller):
 * the k smallest keys of keys[0..n) ascending; ~0 fills when n < k */
int vs_topk_merge_host(const uint64_t* keys, int64_t n, int32_t k, uint64_t* out);
/* filter_poses on bare scores (dock.cpp:373-390) */
int vs_filter_poses(const double* scores, int32_t n, int64_t keep_top, double min_score,
                    int32_t* out_idx);
/* rank_ligands (pipeline.cpp:243-251): ids NUL-separated */
int vs_rank_ligands(const char* ids_blob, const double* scores, int32_t n, int32_t* out_order);
/* id_rank[i] = rank of id i in std::map (bytewise) order */
int vs_id_ranks(const char* ids_blob, int32_t n, uint32_t* out_rank);

#ifdef __cplusplus
}
#endif

#endif /* VSCREEN_GPU_CAPI_H */
