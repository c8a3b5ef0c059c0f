/* gmds.h -- C-ABI of libgmds, the B200 (sm_100a) Gini-MDS hot-path engine.
 *
 * This is the drop-in boundary beneath the ginimds:: C++ facade
 * (include/ginimds/ headers).  Plain pointers and sizes only; no CUDA or torch
 * types.  Every entry point replaces one reference function, cited as
 * /root/reference/proj/core/<file>:<line>.  Host pointers are caller-owned;
 * device handles (gmds_dmat) are library-owned.  Functions are re-entrant;
 * failures return a status mirroring the reference exception classes
 * (error.hpp:9-53) and set a thread-local message (gmds_last_error()).
 *
 * Matrix layout: X is n x p.  GMDS_COL_MAJOR is Eigen's default (the
 * reference's Matrix = Eigen::MatrixXd); distance matrices are symmetric, so
 * their row- and column-major images coincide.
 */
#ifndef GMDS_H
#define GMDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gmds_status {
  GMDS_OK = 0,
  GMDS_INVALID_INPUT = 1,    /* ginimds::InvalidInput    (error.hpp:16-19) */
  GMDS_INVALID_CONFIG = 2,   /* ginimds::InvalidConfig   (error.hpp:22-25) */
  GMDS_DEGENERATE_INPUT = 3, /* ginimds::DegenerateInput (error.hpp:29-32) */
  GMDS_NUMERIC_FAILURE = 4,  /* ginimds::NumericFailure  (error.hpp:35-38) */
  GMDS_ERROR = 5,            /* ginimds::Error (other)                     */
  GMDS_CUDA_ERROR = 6,       /* device failure (no reference counterpart)  */
  GMDS_NCCL_ERROR = 7
} gmds_status;

typedef enum gmds_dtype { GMDS_F32 = 0, GMDS_F64 = 1 } gmds_dtype;
typedef enum gmds_layout { GMDS_ROW_MAJOR = 0, GMDS_COL_MAJOR = 1 } gmds_layout;

/* StressKind, embed.hpp:13 (same order). */
typedef enum gmds_stress_kind { GMDS_KRUSKAL = 0, GMDS_HUBER = 1, GMDS_SAMMON = 2, GMDS_SMACOF = 3 } gmds_stress_kind;
/* EmbeddingMethod, embed.hpp:15 (same order). */
typedef enum gmds_method {
  GMDS_M_CLASSICAL = 0,
  GMDS_M_KRUSKAL = 1,
  GMDS_M_HUBER = 2,
  GMDS_M_SAMMON = 3,
  GMDS_M_SMACOF = 4
} gmds_method;

const char* gmds_last_error(void);
const char* gmds_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host; compute calls then fail with GMDS_CUDA_ERROR). */
int gmds_device_count(void);
gmds_status gmds_set_device(int device);
/* Number of libgmds kernel launches issued by this process so far (bench.py's gpu_launches). */
int64_t gmds_launch_count(void);
/* Make this thread's subsequent calls run on `stream` (a cudaStream_t; NULL
 * restores private per-call streams).  Calls remain blocking. */
gmds_status gmds_set_stream(void* stream);
/* Roofline probe: measured FP32-FMA + INT lane-op rate of this GPU (ops/s). */
gmds_status gmds_probe_alu(double* lane_ops_per_sec);

/* ---- rank: midrank (metrics.hpp:71-72, metrics.cpp:101-110 -> midrank_into 42-56) ----
 * m vectors of length d, row-major (vector k at v + k*d).  ranks: m*d. */
gmds_status gmds_midrank_batch(const double* v, int64_t m, int64_t d, double* ranks);

/* Midranks of z = x_i - x_j (the ranks gen_gini_directed_impl builds,
 * metrics.cpp:69-72, 84-93) for npairs row pairs (pairs[2k], pairs[2k+1]).
 * ranks: npairs*p, in feature order.  Bit-exact verification path. */
gmds_status gmds_pair_midranks(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                               const int64_t* pairs, int64_t npairs, double* ranks);

/* ---- distance: gen_gini_distance (metrics.hpp:105-107, metrics.cpp:157-163) for one pair. */
gmds_status gmds_gen_gini_distance(const double* x, int64_t dx, const double* y, int64_t dy, double nu, double* out);

/* Directed generalized Gini dissimilarity (metrics.hpp:95-97, metrics.cpp:69-93, 148-151). */
gmds_status gmds_gen_gini_directed(const double* x, int64_t dx, const double* y, int64_t dy, double nu, double* out);
/* gini_norm (metrics.hpp:79-80, metrics.cpp:58-66, 112-115). */
gmds_status gmds_gini_norm(const double* x, int64_t d, double* out);
/* gini_pseudo_distance (metrics.hpp:85-86, metrics.cpp:119-127). */
gmds_status gmds_gini_pseudo_distance(const double* x, int64_t dx, const double* y, int64_t dy, double* out);
/* empirical_survival (metrics.hpp:89-90, metrics.cpp:133-144): out[d]. */
gmds_status gmds_empirical_survival(const double* z, int64_t d, double* out);

/* ---- pairwise_matrix, Gini branch (metrics.hpp:112, metrics.cpp:193-219 + from_matrix 169-191).
 * nnu values of nu at once (one sort per pair serves them all).  D: host,
 * nnu consecutive n x n matrices of out_t.  Each nu must be > 1
 * (GiniParams, metrics.hpp:35-36). */
gmds_status gmds_pairwise_gini(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                               const double* nus, int32_t nnu, gmds_dtype out_t, void* D);

/* pairwise_matrix, Euclidean branch (metrics.cpp:220-235).  D: host n x n fp64.
 * n >= 512: tcgen05 path (see gmds_pairwise_euclidean_device), within 1e-6
 * max-normalised of the reference; smaller n: the reference's arithmetic exactly. */
gmds_status gmds_pairwise_euclidean(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, double* D);

/* The Euclidean branch on the device: dX row-major, dD n x n fp64.  mode 0: the
 * tcgen05 path for n >= 512 (bf16x3 split Gram GEMM in TMEM + fp64 norm
 * corrections, near-duplicates recomputed exactly), else the exact fp64 kernel;
 * 1: exact kernel; 2: tcgen05 path. */
gmds_status gmds_pairwise_euclidean_device(const void* dX, gmds_dtype xt, int64_t n, int64_t p, double* dD,
                                           int32_t mode, void* stream);

/* Device-resident variant for callers that keep X and D in HBM (bench,
 * the fit path).  dX row-major on the device; dD receives nnu full n x n
 * matrices (out_t; shard 0 zeroes the diagonal) or, with packed != 0, nnu
 * packed upper-triangle tile
 * images (see gmds_packed_elems).  stream: a cudaStream_t or NULL.
 * shard/nshards split the tile list (multi-GPU, one process per GPU): a
 * shard writes only its own tiles. */
gmds_status gmds_pairwise_gini_device(const void* dX, gmds_dtype xt, int64_t n, int64_t p, const double* nus,
                                      int32_t nnu, gmds_dtype out_t, int32_t packed, void* dD, int32_t shard,
                                      int32_t nshards, void* stream);
/* Elements in one packed upper-triangle image of an n x n matrix. */
int64_t gmds_packed_elems(int64_t n);

/* ---- DistanceMatrix on the device (metrics.hpp:45-57) ---- */
typedef struct gmds_dmat gmds_dmat;
/* DistanceMatrix::from_matrix (metrics.cpp:169-191): validates a host n x n
 * matrix (square, zero diagonal, symmetric to 1e-12 * max(scale,1),
 * finite, non-negative), clamps, uploads in `storage` precision. */
gmds_status gmds_dmat_from_host(const double* D, int64_t n, gmds_dtype storage, gmds_dmat** out);
/* pairwise_matrix(X, gini(nu)) straight into a device handle (no host D). */
gmds_status gmds_dmat_gini(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, double nu,
                           gmds_dtype storage, gmds_dmat** out);
/* Same, from a device-resident row-major X (bench / large n). */
gmds_status gmds_dmat_gini_device(const void* dX, gmds_dtype xt, int64_t n, int64_t p, double nu, gmds_dtype storage,
                                  gmds_dmat** out);
gmds_status gmds_dmat_download(const gmds_dmat* d, double* D_full);
int64_t gmds_dmat_n(const gmds_dmat* d);
void gmds_dmat_free(gmds_dmat* d);

/* ---- stress (embed.hpp:61-76, embed.cpp:111-212, 462-489) ----
 * coords: host n x q column-major (Eigen layout).  huber_delta: NaN = unset
 * (StressConfig::huber_delta empty).  weights: host n x n or NULL (uniform). */
gmds_status gmds_kruskal_stress(const gmds_dmat* D, const double* coords, int32_t q, double* out);
gmds_status gmds_stress_loss(int32_t kind, const gmds_dmat* D, const double* coords, int32_t q, double huber_delta,
                             const double* weights, double* out);
gmds_status gmds_stress_gradient(int32_t kind, const gmds_dmat* D, const double* coords, int32_t q,
                                 double huber_delta, const double* weights, double* grad);

/* One rank's share of a sharded stress pass: raw loss and raw
 * per-row gradient sums of `kind` at coords over this shard's tiles of D
 * (chunks split evenly by block count).  Summing raw_loss / raw_grad over
 * shards 0..nshards-1 (an all-reduce) gives the full pass; the kind's global
 * scale (1/(KS*den) for kruskal, 2/sum(D) for sammon) is applied after the
 * reduction.  q <= 4.  kind GMDS_SMACOF+1 (= 4) is the Guttman transform sum. */
gmds_status gmds_stress_partial(int32_t kind, const gmds_dmat* D, const double* coords, int32_t q, double huber_delta,
                                int32_t shard, int32_t nshards, double* raw_loss, double* raw_grad);
/* Per-fit constants of a device DistanceMatrix: sum D^2, sum D, min and max off-diagonal entry (4 doubles). */
gmds_status gmds_dmat_stats(const gmds_dmat* d, double* stats4);

/* double_center (embed.hpp:51, embed.cpp:382-413): S, B host n x n column-major. */
gmds_status gmds_double_center(const double* S, int64_t n, double* B);

/* classical_mds (embed.cpp:415-460): coords n x q column-major, eigvals q. */
gmds_status gmds_classical_mds(const gmds_dmat* D, int32_t q, double* coords, double* eigvals, int32_t* clamped_count,
                               double* clamped_mass, double* stress);

/* classical_mds, top-q only: the q largest eigenpairs of the
 * double-centred Gram matrix by device subspace iteration (cuBLAS DGEMM on the
 * dense B, Rayleigh-Ritz), same sign rule and clamp as gmds_classical_mds but
 * without the full spectrum (no clamped_mass).  Converged when every top-q
 * residual ||B u - theta u|| <= tol * max|theta|.  GMDS_NUMERIC_FAILURE when
 * not converged in max_iters or when the top q are not separated from the
 * rest of the spectrum.  minimize_stress's classical init uses it for
 * n > 4096.  iterations may be NULL. */
gmds_status gmds_classical_mds_topq(const gmds_dmat* D, int32_t q, double tol, int32_t max_iters, double* coords,
                                    double* eigvals, int32_t* clamped_count, int32_t* iterations);

/* StressConfig (embed.hpp:19-29). */
typedef struct gmds_stress_cfg {
  int32_t kind;         /* gmds_stress_kind */
  double huber_delta;   /* NaN = auto (median grid, embed.cpp:499-515) */
  const double* smacof_weights; /* host n x n or NULL */
  int32_t max_iters;
  double rel_tol;
  uint64_t seed;
} gmds_stress_cfg;

typedef struct gmds_fit_result {
  double* coords;        /* caller buffer n x q column-major */
  double* history;       /* caller buffer, history_cap entries (may be NULL) */
  int64_t history_cap;
  int64_t history_len;   /* out: full length of stress_history */
  int32_t iterations;    /* out */
  int32_t converged;     /* out */
  double stress;         /* out */
  double huber_delta;    /* out: resolved delta when kind == huber */
  int64_t passes;        /* out: device passes over D (observability) */
} gmds_fit_result;

/* minimize_stress (embed.cpp:491-532).  Y0 == NULL starts from
 * classical_mds(D, q) exactly as the reference; a non-NULL Y0 (n x q
 * column-major) is the seeded-init mode. */
gmds_status gmds_minimize_stress(const gmds_dmat* D, int32_t q, const gmds_stress_cfg* cfg, const double* Y0,
                                 gmds_fit_result* res);

/* ---- tune (tune.hpp:42-56, tune.cpp:85-167) ----
 * X host (layout lx) n x p.  grid: m strictly increasing nu > 1.
 * mean_stress: m.  coords: n x q column-major (best / final embedding). */
gmds_status gmds_tune_nu(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                         const double* grid, int32_t m, int32_t k_folds, int32_t method, uint64_t seed,
                         double* mean_stress, double* nu_star, double* coords, double* stress);
/* The whole Embedding (embed.hpp:28-40) a tune entry returns: embed_distances'
 * result (tune.cpp:20-33) -- classical_mds (eigenvalues, clamped stats) or
 * minimize_stress with a default StressConfig (iterations, converged, history,
 * huber_delta).  Caller buffers: coords n x q column-major, eigenvalues q (may
 * be NULL), history history_cap entries (may be NULL). */
typedef struct gmds_embedding {
  double* coords;
  double* eigenvalues;
  double* history;
  int64_t history_cap;
  int64_t history_len;     /* out: full length of stress_history */
  int32_t method;          /* out: gmds_method */
  int32_t n_eigenvalues;   /* out: q for classical, 0 for stress fits (the reference leaves them empty) */
  int32_t clamped_count;   /* out */
  int32_t iterations;      /* out */
  int32_t converged;       /* out */
  double clamped_mass;     /* out */
  double stress;           /* out */
  double huber_delta;      /* out */
} gmds_embedding;
/* tune_nu with TuneReport::best_embedding in full (tune.cpp:132-133). */
gmds_status gmds_tune_nu_ex(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                            const double* grid, int32_t m, int32_t k_folds, int32_t method, uint64_t seed,
                            double* mean_stress, double* nu_star, gmds_embedding* best);
/* alternating_tune with AlternatingResult::embedding in full (tune.cpp:149). */
gmds_status gmds_alternating_tune_ex(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                                     int32_t outer_iters, const double* grid, int32_t m, uint64_t seed,
                                     double* nu_path, double* nu_star, gmds_embedding* emb);
/* Fused nu-sweep scorer (the grid sweep of alternating_tune,
 * tune.cpp:153-157): ks[g] = kruskal_stress(Y, pairwise_matrix(X, gini(grid[g])))
 * for every grid value from ONE distance pass (one sort per pair serves every
 * nu; no D_nu is materialised).  Y host n x q column-major. */
gmds_status gmds_nu_sweep_kruskal(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                                  const double* Y, int32_t q, const double* grid, int32_t m, double* ks);
gmds_status gmds_alternating_tune(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                                  int32_t outer_iters, const double* grid, int32_t m, uint64_t seed, double* nu_path,
                                  double* nu_star, double* coords, double* stress);

/* ---- multi-GPU: one rank per GPU ----
 * The reference's only parallelism is std::thread parallel_for
 * (parallel.hpp:24-59) over rows (metrics.cpp:213-219), (nu, fold) cells
 * (tune.cpp:101-113) and the grid sweep (tune.cpp:154-157); its stress loop
 * is serial (embed.cpp:222-272).  Here the rows of D (its packed blocks) and
 * the nu grid are split across ranks, and the stress iteration is one
 * all-reduce of [gradient | loss sums] per pass, enqueued on the rank's stream
 * (NCCL over NVLink / NVSwitch). */
typedef struct gmds_comm gmds_comm;
#define GMDS_COMM_ID_BYTES 128
/* A new NCCL unique id (rank 0 creates it; the caller's plumbing shares it). */
gmds_status gmds_comm_unique_id(unsigned char* id);
/* Rank `rank` of `nranks` on the current device (gmds_set_device first). */
gmds_status gmds_comm_init_nccl(const unsigned char* id, int32_t nranks, int32_t rank, gmds_comm** out);
/* nranks ranks in ONE process on the current device (tests with fewer GPUs
 * than ranks): comms[r] must be driven by its own host thread; collectives are
 * one reduction kernel over every rank's buffer in rank order. */
gmds_status gmds_comm_init_local(int32_t nranks, gmds_comm** comms);
int32_t gmds_comm_rank(const gmds_comm* c);
int32_t gmds_comm_size(const gmds_comm* c);
/* In-place all-reduce of a device buffer (op 0 sum, 1 min, 2 max); blocking. */
gmds_status gmds_comm_allreduce_device(gmds_comm* c, double* dbuf, int64_t count, int32_t op, void* stream);
void gmds_comm_free(gmds_comm* c);

/* This rank's share of pairwise_matrix(X, gini(nu)) kept on the device: the
 * contiguous range [nblk*r/N, nblk*(r+1)/N) of the packed 128 x 128 blocks
 * (row-major upper triangle), computed here and nowhere else; the per-fit
 * constants (sum D^2, sum D, min, max) are all-reduced over the group.  dX:
 * the full row-major X on this device.  Usable by gmds_minimize_stress_sharded
 * and gmds_dmat_stats only. */
gmds_status gmds_dmat_gini_sharded(gmds_comm* comm, const void* dX, gmds_dtype xt, int64_t n, int64_t p, double nu,
                                   gmds_dtype storage, gmds_dmat** out);
/* minimize_stress (embed.cpp:491-532) over a row-sharded D: every rank runs
 * the device-resident loop on its blocks and all-reduces [gradient | loss sums]
 * once per pass; every rank returns the same embedding.  fp32 storage, q <= 4,
 * seeded start Y0 (n x q column-major, required: the classical init needs all of
 * D), Huber with an explicit delta. */
gmds_status gmds_minimize_stress_sharded(gmds_comm* comm, const gmds_dmat* D, int32_t q, const gmds_stress_cfg* cfg,
                                         const double* Y0, gmds_fit_result* res);
/* The fused nu-sweep scorer over a nu grid split across ranks (tune.cpp:153-157
 * with the grid shared out as replicas): each rank scores its contiguous block of
 * grid values from one distance pass, the scores are all-reduced, and every rank
 * returns all m values.  X, Y host as gmds_nu_sweep_kruskal. */
gmds_status gmds_nu_sweep_kruskal_sharded(gmds_comm* comm, const void* X, gmds_dtype xt, gmds_layout lx, int64_t n,
                                          int64_t p, const double* Y, int32_t q, const double* grid, int32_t m,
                                          double* ks);

#ifdef __cplusplus
}
#endif

#endif /* GMDS_H */
