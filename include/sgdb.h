/*
 * sgdb.h — C-ABI of the B200-native GLM SGD engine (libsgdb_b200.so).
 *
 * Drop-in boundary for the reference's training path. The reference
 * (/root/reference/proj, C++20, CPU-only) exposes no FFI: its boundary is the
 * C++ API in proj/include/sgdbench/{sync_engine,async_engine,linalg,glm,
 * dataset,fixtures}.hpp, called by harness::run_engine_once
 * (proj/src/harness.cpp:75-124). This header re-expresses that API as plain C
 * (opaque handles, plain pointers and sizes, integer status codes) so that the
 * C++ host engine in this library, a C++ adapter for the reference harness
 * (INTEGRATION.md), and Python (ctypes) all bind the same entry points.
 *
 * Layers:
 *   1. device ops    — context, device-resident dataset/model, one sync epoch,
 *                      one Hogwild epoch, replica averaging, loss. Each
 *                      launches hand-written sm_100a kernels.
 *   2. whole runs    — sgdb_sync_train / sgdb_hogwild_train /
 *                      sgdb_numa_dual_train: the reference's epoch loops
 *                      (host C++: schedule, timing, hooks, budget, divergence)
 *                      over layer 1.
 *   3. host helpers  — fixtures, LIBSVM parsing, binary cache, layout
 *                      conversion, worker assignment, plan grammar, the
 *                      mini-batch schedule. Pure host code, no GPU needed.
 *
 * Errors: every function returns sgdb_status; on failure
 * sgdb_last_error() (thread-local) holds the message. The codes map 1:1 onto
 * the reference's exception types (std::invalid_argument, std::domain_error,
 * ParseError, CapacityError, std::runtime_error). Divergence is NOT an error:
 * it is reported in-band in sgdb_trace, as LossTrace does
 * (proj/src/sync_engine.cpp:107-113).
 *
 * Precision: the interface is fp64 like the reference (dataset.hpp:46-48);
 * by default device storage and per-example arithmetic are fp32, reductions
 * and the synchronous master model fp64. Datasets
 * uploaded with SGDB_UPLOAD_EXACT_FP64 run every op in fp64 in the
 * reference's operation order instead (bit-identical results).
 */
#ifndef SGDB_H_
#define SGDB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
typedef int32_t sgdb_status;
#define SGDB_OK 0
#define SGDB_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument           */
#define SGDB_ERR_DOMAIN 2           /* std::domain_error                */
#define SGDB_ERR_PARSE 3            /* sgdbench::ParseError (dataset.hpp:22-26) */
#define SGDB_ERR_CAPACITY 4         /* sgdbench::CapacityError (dataset.hpp:28-30) */
#define SGDB_ERR_RUNTIME 5          /* std::runtime_error (I/O)         */
#define SGDB_ERR_CUDA 6             /* CUDA runtime / launch failure    */
#define SGDB_ERR_UNSUPPORTED 7      /* plan/layout combination not built on the device */

/* ---- enums (same numbering as the reference enums) ---------------------- */
typedef enum { SGDB_TASK_LR = 0, SGDB_TASK_SVM = 1 } sgdb_task;           /* glm.hpp:15 */
typedef enum {                                                             /* dataset.hpp:13 */
  SGDB_LAYOUT_DENSE_ROW = 0,
  SGDB_LAYOUT_DENSE_COL = 1,
  SGDB_LAYOUT_CSR = 2,
  SGDB_LAYOUT_PADDED = 3
} sgdb_layout;
typedef enum { SGDB_STRATEGY_ROUND_ROBIN = 0, SGDB_STRATEGY_CHUNK = 1 } sgdb_strategy; /* dataset.hpp:133 */
typedef enum {                                                             /* async_engine.hpp:17 */
  SGDB_ACCESS_ROW_RR = 0,
  SGDB_ACCESS_ROW_CH = 1,
  SGDB_ACCESS_COL_RR = 2,
  SGDB_ACCESS_COL_CH = 3
} sgdb_access_path;
typedef enum {                                                             /* async_engine.hpp:21 */
  SGDB_REPL_KERNEL = 0,
  SGDB_REPL_BLOCK = 1,
  SGDB_REPL_THREAD = 2,
  SGDB_REPL_EXAMPLE = 3
} sgdb_replication;
typedef enum {                                                             /* linalg.hpp:40 */
  SGDB_EW_MUL = 0,
  SGDB_EW_DIV = 1,
  SGDB_EW_EXP = 2,
  SGDB_EW_NEG = 3,
  SGDB_EW_ADD_SCALAR = 4,
  SGDB_EW_SIGMOID = 5,          /* ew_sigmoid (linalg.hpp:47), not in the reference enum */
  SGDB_EW_HINGE_INDICATOR = 6   /* ew_hinge_indicator (linalg.hpp:50) */
} sgdb_elementwise_op;

/* ---- plain structs ------------------------------------------------------- */

/* Borrowed host view of a dataset; field-for-field sgdbench::Dataset
 * (dataset.hpp:42-61). row_offsets is size_t in the reference: uint64 here. */
typedef struct sgdb_dataset_view {
  uint64_t n_examples;
  uint64_t n_features;
  int32_t layout; /* sgdb_layout */
  const double* labels;         /* n_examples, each +1/-1 */
  const double* values;         /* n_values */
  uint64_t n_values;
  const uint32_t* indices;      /* n_indices (Csr / PaddedDense) */
  uint64_t n_indices;
  const uint64_t* row_offsets;  /* n_examples + 1 (Csr) */
  uint64_t n_row_offsets;
  uint64_t padded_width;        /* PaddedDense */
} sgdb_dataset_view;

/* Hyperparams (glm.hpp:22-35). step_size(e) = alpha * step_decay^(e-1). */
typedef struct sgdb_hyperparams {
  double alpha;
  uint64_t batch_b;
  uint64_t epochs;
  int32_t task; /* sgdb_task */
  double step_decay;
} sgdb_hyperparams;

/* ExecutionPlan (async_engine.hpp:25-33). On the device a "worker" is a lane
 * group (one warp by default) walking its assign()
 * list; workers, group_size, k keep the reference's meaning. */
typedef struct sgdb_plan {
  int32_t access_path; /* sgdb_access_path */
  int32_t replication; /* sgdb_replication */
  uint64_t data_replication_k;
  uint64_t workers;
  uint64_t group_size;
  int32_t circular_offsets;
  uint64_t merge_period_epochs;
  int32_t lanes_per_worker; /* device-only knob: 0 = auto, else 1/2/4/8/16/32 */
} sgdb_plan;

/* EpochRecord (trace.hpp:21-25). */
typedef struct sgdb_epoch_record {
  uint64_t epoch; /* 1-based */
  double loss;
  double seconds; /* compute-only, loss evaluation excluded */
} sgdb_epoch_record;

/* LossTrace (trace.hpp:27-49) + Result::evals_per_epoch (async_engine.hpp:84-88).
 * The caller owns the arrays; capacity bounds both. */
typedef struct sgdb_trace {
  sgdb_epoch_record* epochs;
  uint64_t* evals_per_epoch; /* may be NULL; Hogwild only */
  uint64_t capacity;
  uint64_t count;
  int32_t diverged;
  char divergence_note[160];
} sgdb_trace;

typedef double (*sgdb_clock_fn)(void* user);                               /* Clock (trace.hpp:14-19) */
typedef void (*sgdb_epoch_hook_fn)(void* user, uint64_t epoch, double loss);

/* TrainOptions (sync_engine.hpp:15-25) / hogwild::Options (async_engine.hpp:77-82). */
typedef struct sgdb_train_options {
  uint32_t workers; /* accepted for signature parity; the device ignores it */
  int32_t shuffle;  /* sync only */
  double max_seconds;
  const double* initial_model; /* NULL or n_features doubles */
  uint64_t initial_model_len;
  sgdb_clock_fn clock;        /* NULL = steady clock */
  void* clock_user;
  sgdb_epoch_hook_fn epoch_hook; /* NULL = none */
  void* hook_user;
} sgdb_train_options;

/* Collective hook for multi-GPU runs: called by the engine at each exchange
 * step with a device buffer to SUM-reduce in place across ranks on `stream`
 * (dtype 0 = float32, 1 = float64), for hosts that bring their own process
 * group. The engine can also own an NCCL communicator (sgdb_ctx_init_nccl),
 * which takes precedence. */
typedef int32_t (*sgdb_allreduce_fn)(void* user, void* device_buffer, uint64_t count,
                                     int32_t dtype, void* stream);

/* ---- opaque handles ------------------------------------------------------ */
typedef struct sgdb_ctx sgdb_ctx;
typedef struct sgdb_dataset sgdb_dataset;           /* device-resident */
typedef struct sgdb_model sgdb_model;               /* device-resident */
typedef struct sgdb_host_dataset sgdb_host_dataset; /* library-owned host arrays */
typedef struct sgdb_schedule sgdb_schedule;

/* ======================================================================== */
/* 1. device ops                                                            */
/* ======================================================================== */

const char* sgdb_last_error(void);
const char* sgdb_version(void);

/* Device context: device ordinal + the CUDA stream every op is queued on
 * (NULL = the context creates its own). One host thread per context. */
sgdb_status sgdb_ctx_create(int32_t device, void* cuda_stream, sgdb_ctx** out);
sgdb_status sgdb_ctx_destroy(sgdb_ctx* ctx);
sgdb_status sgdb_ctx_stream(sgdb_ctx* ctx, void** stream_out);
sgdb_status sgdb_ctx_synchronize(sgdb_ctx* ctx);
/* Number of this library's kernels launched on the context so far. */
sgdb_status sgdb_ctx_launch_count(sgdb_ctx* ctx, uint64_t* out);
sgdb_status sgdb_ctx_set_allreduce(sgdb_ctx* ctx, sgdb_allreduce_fn fn, void* user);
/* In-library NCCL communicator (multi-GPU without a host collective
 * provider; generalises numa_dual_train's replica exchange,
 * proj/src/async_engine.cpp:462-520, to G GPUs). Rank 0 creates the 128-byte
 * id, the host distributes it (any channel), every rank attaches its context.
 * The engine then SUM-reduces gradients / models / losses with ncclAllReduce
 * on the context stream — mini-batch steps stay CUDA-graph-replayed. NCCL is
 * resolved at run time (libnccl.so.2); absent -> SGDB_ERR_RUNTIME. */
sgdb_status sgdb_nccl_get_unique_id(uint8_t* id_out /* 128 bytes */);
sgdb_status sgdb_ctx_init_nccl(sgdb_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id);
sgdb_status sgdb_ctx_world(sgdb_ctx* ctx, int32_t* rank, int32_t* nranks);
/* Per-launch CUDA-event timing of this library's kernels on the context
 * stream (off by default; enabling clears earlier records). Entry i of the
 * per-kernel aggregate: name, launches, total milliseconds; *n_entries is the
 * number of distinct kernels. */
sgdb_status sgdb_ctx_set_profiling(sgdb_ctx* ctx, int32_t enable);
sgdb_status sgdb_ctx_kernel_stats(sgdb_ctx* ctx, uint64_t i, char* name, uint64_t cap,
                                  uint64_t* launches, double* total_ms, uint64_t* n_entries);
/* Worker geometry the Hogwild kernels resolve for `lanes` lanes per worker
 * (0 = auto for this dataset): the number of concurrently resident workers. */
sgdb_status sgdb_ctx_resident_workers(sgdb_ctx* ctx, const sgdb_dataset* ds,
                                      int32_t lanes_per_worker, uint64_t* out);

/* Upload (untimed setup): fp64 host values -> fp32 device
 * storage. Dense layouts are stored row-major, PaddedDense/Csr as CSR (plus
 * the original slot-major padded arrays for the column access paths).
 * row_base / n_global describe a row shard of a larger logical dataset
 * (multi-GPU); pass 0 / n_examples for a whole dataset. */
sgdb_status sgdb_dataset_upload(sgdb_ctx* ctx, const sgdb_dataset_view* view, uint64_t row_base,
                                uint64_t n_global, sgdb_dataset** out);
/* Upload with flags. SGDB_UPLOAD_EXACT_FP64 also keeps the fp64 values and
 * switches every op on the dataset to the exact-fp64 mode: sync epochs,
 * batch_gradient and epoch_batch run the reference's primitive chain in its
 * summation order, Hogwild runs process_examples in fp64 (bit-identical with
 * one worker), the loss sums in id order, and exp is glibc's, restated
 * (kernels_linalg.cu, libm_exp.hpp). Results then equal the reference's bit
 * for bit (LR losses to the ulp of log1p). Whole (unsharded) datasets only. */
#define SGDB_UPLOAD_EXACT_FP64 1u
/* SGDB_UPLOAD_PADDED: a CSR view is uploaded and its slot-major padded copy
 * (convert_layout(Csr -> PaddedDense), proj/src/dataset.cpp:380-402: width =
 * the longest row, sentinel index d with value 0) is built on the device; the
 * dataset then behaves as a PaddedDense upload (column access paths). */
#define SGDB_UPLOAD_PADDED 2u
sgdb_status sgdb_dataset_upload_ex(sgdb_ctx* ctx, const sgdb_dataset_view* view, uint64_t row_base,
                                   uint64_t n_global, uint32_t flags, sgdb_dataset** out);
/* Re-copy host arrays of the same shape into an existing device dataset
 * (the e2e leg of bench.py): fp32 values/labels straight from (pinned) host
 * buffers, asynchronously on the context stream. indices/row_offsets may be
 * NULL to keep the device copies. Refreshing a CSR dataset's values, indices
 * or row offsets drops its row-blocked CSC copy: Hogwild and mini-batch sync
 * keep working, full-batch sync then returns SGDB_ERR_UNSUPPORTED (upload
 * again to rebuild it). */
sgdb_status sgdb_dataset_refresh_f32(sgdb_ctx* ctx, sgdb_dataset* ds, const float* values,
                                     const float* labels, const uint32_t* indices,
                                     const uint32_t* row_offsets32);
/* Compact transfer of the column ids of a CSR dataset with d <= 65536: nnz
 * 16-bit ids copied host -> device on ctx's stream and widened there to the
 * 32-bit ids the kernels read (half the index bytes over PCIe). Same
 * invalidation as sgdb_dataset_refresh_f32. Not in the reference API (its
 * datasets live in host memory); it serves hosts that stream inputs. */
sgdb_status sgdb_dataset_refresh_idx16(sgdb_ctx* ctx, sgdb_dataset* ds, const uint16_t* indices16);
sgdb_status sgdb_dataset_free(sgdb_dataset* ds);
/* K9: generate a dense synthetic classification shard on the device (rows
 * [row_base, row_base + n_local) of an n_global x d dataset) — the
 * distribution of fixtures::dense_classification (fixtures.cpp:30-52) with a
 * counter-based Philox-4x32-10 stream, so the 200M x 1000 configuration can
 * be produced where it is trained and any slice re-created on the CPU
 * (oracle/glm_oracle.cpp orc_philox_dense). 1 <= d <= 1024. */
sgdb_status sgdb_dataset_generate_dense(sgdb_ctx* ctx, uint64_t n_local, uint64_t d,
                                        uint64_t row_base, uint64_t n_global, uint64_t seed,
                                        double label_noise, sgdb_dataset** out);
/* Copy rows [row0, row0+nrows) of a dense device dataset back (fp32). */
sgdb_status sgdb_dataset_read_dense(sgdb_ctx* ctx, const sgdb_dataset* ds, uint64_t row0,
                                    uint64_t nrows, float* values_out, float* labels_out);
/* The generator's hidden model w_true (Box-Muller over Philox; host). */
sgdb_status sgdb_generate_hidden_model(uint64_t seed, uint64_t d, double* out);
/* Algorithmic bytes of one sweep: CSR nnz*8 + (N+1)*4 + N*4;
 * dense N*d*4 + N*4. */
sgdb_status sgdb_dataset_sweep_bytes(const sgdb_dataset* ds, uint64_t* out);
sgdb_status sgdb_dataset_shape(const sgdb_dataset* ds, uint64_t* n_local, uint64_t* d,
                               uint64_t* nnz, uint64_t* row_base, uint64_t* n_global);

sgdb_status sgdb_model_create(sgdb_ctx* ctx, uint64_t d, const double* init, sgdb_model** out);
sgdb_status sgdb_model_set(sgdb_ctx* ctx, sgdb_model* m, const double* w);
sgdb_status sgdb_model_get(sgdb_ctx* ctx, sgdb_model* m, double* w_out);
/* Device pointers of the fp32 working copy (d+1 floats, guard slot d == 0)
 * and of the fp64 master (d doubles). */
sgdb_status sgdb_model_device_ptrs(sgdb_model* m, float** w32, double** w64);
sgdb_status sgdb_model_free(sgdb_model* m);

/* One synchronous epoch (sync_engine.cpp:86-100): the ids in `order`
 * (host; NULL = ascending 0..n_global-1) taken as consecutive mini-batches of
 * batch_b; per batch g = X_B^T c(X_B w) then w -= alpha*g. With
 * batch_b >= n_global the epoch is one full-batch step and `order` is not
 * read. *finite_out = 0 if any gradient entry was non-finite (the epoch stops
 * after that batch, as the reference does); passing finite_out == NULL makes
 * the call fully asynchronous on the context stream. */
sgdb_status sgdb_sync_epoch(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                            double alpha, const uint32_t* order, uint64_t batch_b,
                            int32_t* finite_out);
/* sync::batch_gradient (sync_engine.hpp:33-36): g over `rows` (global ids;
 * n_rows == 0 = all) at the host model w. No update. `transposed` != 0 says
 * the caller would pass the materialised column-major transpose: in the
 * exact-fp64 mode it selects the per-column summation order for dense data. */
sgdb_status sgdb_batch_gradient(sgdb_ctx* ctx, sgdb_dataset* ds, int32_t task,
                                const uint32_t* rows, uint64_t n_rows, const double* w,
                                int32_t transposed, double* g_out);
/* sync::epoch_batch (sync_engine.hpp:40-41): one B=N step, returns ||g||_2. */
sgdb_status sgdb_epoch_batch(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                             double alpha, double* grad_norm_out);

/* One Hogwild epoch of `plan` (async_engine.cpp:244-254 + 372-396): replica
 * prepare, the workers' passes, replica merge. *evals_out = n + T_nonempty*k.
 * Asynchronous on the context stream (like a kernel launch): synchronise, or
 * read the model, before using results on the host. */
sgdb_status sgdb_hogwild_epoch(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                               double alpha, const sgdb_plan* plan, uint64_t* evals_out);
/* Segment seg of nseg of that epoch: every worker runs positions
 * [t*seg/nseg, t*(seg+1)/nseg) of its assign() list (t = its length), with
 * replica prepare/merge around it. Running segments 0..nseg-1 back to back
 * is one epoch with a barrier after each segment; the multi-GPU Hogwild
 * path averages the rank replicas at those barriers (the
 * numa_dual_train merge, async_engine.cpp:478-501, made k times per epoch).
 * *evals_out = evaluations in this segment. */
sgdb_status sgdb_hogwild_segment(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                                 double alpha, const sgdb_plan* plan, uint32_t seg, uint32_t nseg,
                                 uint64_t* evals_out);
/* merge_models (async_engine.cpp:133-156) over device models: out = weighted
 * mean (weights NULL = unweighted); when refresh != 0 every input is set to it. */
sgdb_status sgdb_models_average(sgdb_ctx* ctx, sgdb_model* const* models, uint64_t count,
                                const double* weights, sgdb_model* out, int32_t refresh);

/* Multi-GPU replica averaging (the numa_dual_train merge generalised to G
 * ranks, async_engine.cpp:478-501): SUM all-reduce of the fp64 model through
 * the context's hook, then scale by 1/world. */
sgdb_status sgdb_model_average_ranks(sgdb_ctx* ctx, sgdb_model* m, uint64_t world);

/* dataset_loss (glm.cpp:85-94): sum of point losses, fp64. With an allreduce
 * hook set the per-shard sum is reduced across ranks. */
sgdb_status sgdb_loss(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                      double* loss_out);

/* ---- the §4 operator API (linalg.hpp:23-58) ------------------------------
 * Stand-alone device primitives with host vectors in and out (the training
 * path uses the fused kernels instead). fp64 arithmetic on the uploaded fp32
 * matrix, with the reference's summation order: matvec sums each row in slot
 * order; matvec_transposed is one sequential dot per column for a
 * DenseColMajor upload and 256-row block partials + the fixed pairwise tree
 * otherwise (linalg.cpp:46-109), so results equal the reference on the same
 * (f32-valued) matrix. rows NULL / n_rows 0 = all examples (ascending). */
sgdb_status sgdb_matvec(sgdb_ctx* ctx, sgdb_dataset* ds, const uint32_t* rows, uint64_t n_rows,
                        const double* v, uint64_t v_len, double* out /* n_rows or n */);
sgdb_status sgdb_matvec_transposed(sgdb_ctx* ctx, sgdb_dataset* ds, const uint32_t* rows,
                                   uint64_t n_rows, const double* a_by_position, uint64_t a_len,
                                   double* out /* d */);
/* ew_* / elementwise (linalg.hpp:35-55); b is read by MUL and DIV only, scalar
 * by ADD_SCALAR. DIV with a zero divisor -> SGDB_ERR_DOMAIN. */
sgdb_status sgdb_elementwise(sgdb_ctx* ctx, int32_t op, const double* a, const double* b,
                             uint64_t n, double scalar, double* out);
/* axpy (linalg.hpp:58): w <- w - alpha * g, in place on the host array. */
sgdb_status sgdb_axpy(sgdb_ctx* ctx, double* w, double alpha, const double* g, uint64_t n);

/* ======================================================================== */
/* 2. whole runs (host C++ epoch loops over layer 1)                        */
/* ======================================================================== */

/* sync::train (sync_engine.hpp:51-52). */
sgdb_status sgdb_sync_train(sgdb_ctx* ctx, sgdb_dataset* ds, const sgdb_hyperparams* hyper,
                            uint64_t seed, const sgdb_train_options* options, double* model_out,
                            sgdb_trace* trace);
/* hogwild::train (async_engine.hpp:96-97). */
sgdb_status sgdb_hogwild_train(sgdb_ctx* ctx, sgdb_dataset* ds, const sgdb_hyperparams* hyper,
                               const sgdb_plan* plan, uint64_t seed,
                               const sgdb_train_options* options, double* model_out,
                               sgdb_trace* trace);
/* hogwild::numa_dual_train (async_engine.hpp:102-104): two full-data
 * replicas averaged every merge_period_epochs. */
sgdb_status sgdb_numa_dual_train(sgdb_ctx* ctx, sgdb_dataset* ds, const sgdb_hyperparams* hyper,
                                 const sgdb_plan* plan, uint64_t seed,
                                 const sgdb_train_options* options, double* model_out,
                                 sgdb_trace* trace);

/* ======================================================================== */
/* 3. host helpers (no GPU)                                                 */
/* ======================================================================== */

/* fixtures::dense_classification / sparse_classification (fixtures.hpp:12-19). */
sgdb_status sgdb_fixture_dense(uint64_t n, uint64_t d, uint64_t seed, double label_noise,
                               sgdb_host_dataset** out);
sgdb_status sgdb_fixture_sparse(uint64_t n, uint64_t d, double avg_nnz, uint64_t seed,
                                double label_noise, sgdb_host_dataset** out);
/* parse_libsvm (dataset.hpp:101). declared_d < 0 = none. On SGDB_ERR_PARSE
 * *error_line is the 1-based line number. */
sgdb_status sgdb_parse_libsvm(const char* text, uint64_t len, int64_t declared_d,
                              sgdb_host_dataset** out, uint64_t* error_line);
/* write_libsvm (dataset.hpp:104): *len_out = bytes needed; text written when cap suffices. */
sgdb_status sgdb_write_libsvm(const sgdb_dataset_view* view, char* buf, uint64_t cap,
                              uint64_t* len_out);
/* save_binary / load_binary (dataset.hpp:107-109), magic "sgdbds01". */
sgdb_status sgdb_save_binary(const sgdb_dataset_view* view, const char* path);
sgdb_status sgdb_load_binary(const char* path, sgdb_host_dataset** out);
/* convert_layout (dataset.hpp:117-118); max_dense_bytes 0 = 2 GiB default. */
sgdb_status sgdb_convert_layout(const sgdb_dataset_view* view, int32_t target,
                                uint64_t max_dense_bytes, sgdb_host_dataset** out);
/* Dataset::validate (dataset.hpp:56). */
sgdb_status sgdb_validate_dataset(const sgdb_dataset_view* view);
sgdb_status sgdb_host_dataset_view(const sgdb_host_dataset* h, sgdb_dataset_view* out);
sgdb_status sgdb_host_dataset_free(sgdb_host_dataset* h);

/* assign (dataset.hpp:153): lists flattened in worker order; offsets has
 * workers+1 entries. Pass NULL arrays to query *total. */
sgdb_status sgdb_assign(uint64_t n, uint64_t workers, int32_t strategy, uint64_t k,
                        uint32_t* ids_out, uint64_t* offsets_out, uint64_t* total);
/* parse_plan / plan_to_string / validate_plan (async_engine.hpp:40-47).
 * Parsing fills the reference defaults (workers 1, group 32, offsets on,
 * merge period 1, lanes auto). */
sgdb_status sgdb_parse_plan(const char* text, sgdb_plan* out);
sgdb_status sgdb_plan_to_string(const sgdb_plan* plan, char* buf, uint64_t cap);
sgdb_status sgdb_validate_plan(const sgdb_plan* plan, int32_t layout);

/* The mini-batch schedule of sync::train (sync_engine.cpp:75-84):
 * mt19937_64(seed), iota, one std::shuffle per epoch when shuffle != 0. */
sgdb_status sgdb_schedule_create(uint64_t seed, uint64_t n, int32_t shuffle, sgdb_schedule** out);
sgdb_status sgdb_schedule_next(sgdb_schedule* s, uint32_t* order_out);
sgdb_status sgdb_schedule_free(sgdb_schedule* s);

#ifdef __cplusplus
}
#endif

#endif /* SGDB_H_ */
