/*
 * smlrt_b200.h -- C-ABI of the B200-native `ml(infer)` region runtime.
 *
 * This is the boundary a host binding (ctypes here) calls
 * in place of the reference's pure-numpy data path.  Every entry point names
 * the reference function it replaces; all pointers are plain device/host
 * addresses, all sizes plain integers, no torch types.
 *
 * Conventions
 *   - Return value: smlrt_status_t.  On failure smlrt_last_error() gives a
 *     thread-local message.  Codes map 1:1 onto the reference exception
 *     classes (/root/reference/pkg/src/smlrt/errors.py).
 *   - Launches are asynchronous on the caller's cudaStream_t (passed as
 *     void*).  Device-side failures (non-finite output) are reported through
 *     a caller-owned device status word (uint32_t*), read after the stream
 *     synchronises; SMLRT_STATUS_NONFINITE is set when any output row is
 *     NaN/inf.
 *   - Array pointers are borrowed; plans and models are owned handles.
 *   - One thread of control per handle, as in the reference
 *     (runtime.py:22).
 */
#ifndef SMLRT_B200_H
#define SMLRT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMLRT_MAX_SWEEP 6 /* sweep axes of one map (LHS symbols)          */
#define SMLRT_MAX_FEAT 6  /* feature axes of one RHS view                 */

typedef enum {
  SMLRT_OK = 0,
  SMLRT_E_ARITY = 1,        /* ArityMismatchError                        */
  SMLRT_E_OOB = 2,          /* OutOfBoundsError                          */
  SMLRT_E_FEATURE = 3,      /* FeatureMismatchError                      */
  SMLRT_E_SHAPE = 4,        /* ShapeMismatchError                        */
  SMLRT_E_NONINJECTIVE = 5, /* NonInjectiveScatterError                  */
  SMLRT_E_MODEL_SHAPE = 6,  /* ModelShapeMismatchError                   */
  SMLRT_E_NONFINITE = 7,    /* NonFiniteOutputError                      */
  SMLRT_E_CUDA = 8,         /* CUDA runtime failure                      */
  SMLRT_E_INVALID = 9,      /* bad argument (ValueError)                 */
  SMLRT_E_UNSUPPORTED = 10  /* shape/precision combination not built     */
} smlrt_status_t;

typedef enum { SMLRT_F32 = 0, SMLRT_F64 = 1 } smlrt_dtype_t;
typedef enum { SMLRT_TO = 0, SMLRT_FROM = 1 } smlrt_direction_t;
typedef enum { SMLRT_IDENTITY = 0, SMLRT_RELU = 1, SMLRT_TANH = 2 } smlrt_act_t;
typedef enum { SMLRT_FP32_EXACT = 0, SMLRT_BF16 = 1 } smlrt_precision_t;

/* device status word bits */
#define SMLRT_STATUS_NONFINITE 0x1u

/* region flags */
#define SMLRT_COMMIT_FUSED 0x0   /* epilogue writes outputs directly          */
#define SMLRT_COMMIT_CHECKED 0x1 /* stage, check finiteness, then write       */
#define SMLRT_FORCE_UNFUSED 0x2  /* gather -> per-layer -> scatter (diagnostic)*/
#define SMLRT_SYNC_STATUS 0x4    /* reset *d_status first; afterwards copy it   */
                                 /* to host, synchronise the stream and return */
                                 /* SMLRT_E_NONFINITE if it is set (one call,  */
                                 /* one sync: runtime.py:341's raise)           */

/*
 * One RHS view of a tensor functor applied to one array: the flattening of
 * the reference's MemoryView (bridge.py:148-167, built by wrap_tensors
 * bridge.py:288-344).  Element address of (sweep index s, feature index f):
 *   base + sum_k s_k*sweep_stride[k] + sum_a f_a*feat_stride[a]
 * Feature axes flatten row-major; views concatenate along the feature axis
 * in declaration order (compose_tensor, bridge.py:351-381).
 */
typedef struct {
  int32_t array;  /* index into the ptr/dtype arrays passed at launch */
  int32_t n_feat; /* feature axes, >= 1 (a point slice has (1),(1))   */
  int64_t base;
  int64_t sweep_stride[SMLRT_MAX_SWEEP];
  int64_t feat_count[SMLRT_MAX_FEAT];
  int64_t feat_stride[SMLRT_MAX_FEAT];
} smlrt_view_t;

typedef struct smlrt_plan_s* smlrt_plan_t;
typedef struct smlrt_model_s* smlrt_model_t;

typedef struct {
  int64_t n_rows; /* product of the sweep shape                       */
  int32_t n_cols; /* dense feature width                              */
  int32_t n_views;
  int32_t n_arrays;
  int32_t uniform;     /* all views share one array and sweep strides */
  int32_t dense_rows;  /* uniform and columns are one contiguous run   */
  int32_t injective;   /* FROM plans: proven injective                 */
  int64_t row_pitch;   /* dense_rows: element step between rows (1-D)  */
} smlrt_plan_info_t;

typedef enum { SMLRT_DENSE = 0, SMLRT_CONV2D = 1, SMLRT_MAXPOOL2D = 2 } smlrt_layer_kind_t;

/* One layer, host pointers, copied at upload.
 *  DENSE    : weights [out x in] row-major + bias [out] (models.py:40-64).
 *  CONV2D   : non-overlapping (stride == kernel) convolution of an
 *             [in_channels x in_h x in_w] image; weights [out_channels x
 *             in_channels*kernel*kernel] in (c, dy, dx) row-major order, bias
 *             [out_channels]; out = out_channels*(in_h/k)*(in_w/k) flattened
 *             (channel, row, column).  Format extension, SURVEY.md 8(f).
 *  MAXPOOL2D: kernel x kernel max (NaN-propagating), no parameters.
 * `in`/`out` are the flattened widths for every kind. */
typedef struct {
  int32_t kind;       /* smlrt_layer_kind_t */
  int32_t in;
  int32_t out;
  int32_t activation; /* smlrt_act_t */
  int32_t kernel, stride, in_channels, in_h, in_w;
  const float* weights;
  const float* bias;
} smlrt_layer_t;

const char* smlrt_version(void);
const char* smlrt_last_error(void);
/* Number of CUDA kernels this library has launched since it was loaded
 * (instrumentation: the bench reports its own launches per timed region). */
unsigned long long smlrt_launch_count(void);

/*
 * Plan compiler.  Replaces the per-call extract/resolve/wrap + np.unique of
 * the reference (bridge.py:388-395 for TO, bridge.py:407-448 for FROM):
 * validates every flat address against its array's storage (OutOfBounds) and,
 * for FROM plans, proves injectivity once (analytically, else by an exact
 * host bitmap over the destination span) -> NonInjectiveScatter.  Pure host
 * code; device tables are uploaded lazily per device on first launch.
 */
int smlrt_plan_create(const smlrt_view_t* views, int n_views, int n_sweep,
                      const int64_t* sweep_shape, int direction,
                      const int64_t* array_numel, int n_arrays,
                      smlrt_plan_t* out);
int smlrt_plan_info(smlrt_plan_t plan, smlrt_plan_info_t* info);
/* Element ranges [lo, hi) of a uniform 1-D-sweep plan's single array touched
 * by sweep rows [r0, r1): one per column, sorted, overlapping/adjacent ones
 * merged; `ranges` holds 2*max_ranges int64.  *exact = 1 when every element
 * inside the ranges is touched (column stride 1 or dense row-major rows), so
 * the ranges are also safe to copy back for a FROM plan.  Host-side chunking
 * of host-resident arrays (copy a row block's bytes, launch on it). New in
 * this runtime (no reference counterpart). SMLRT_E_UNSUPPORTED if the plan
 * is not uniform / not 1-D or needs more than max_ranges ranges. */
int smlrt_plan_row_ranges(smlrt_plan_t plan, int64_t r0, int64_t r1, int64_t* ranges, int32_t max_ranges,
                          int32_t* n_ranges, int32_t* exact);
int smlrt_plan_destroy(smlrt_plan_t plan);

/*
 * Model upload.  Replaces load_model's in-memory form (models.py:107-151)
 * for the device: weights copied once to `device` in the layout the chosen
 * precision's kernels consume (f32 for FP32_EXACT; bf16 K-major + f32 bias
 * for BF16).  Rejects non-finite parameters (NonFiniteWeightsError is raised
 * by the Python layer before upload).
 */
int smlrt_model_upload(const smlrt_layer_t* layers, int n_layers,
                       int precision, int device, smlrt_model_t* out);
int smlrt_model_free(smlrt_model_t model);
/* which kernel region_infer would run: 0 none, 1 fused exact (templated),
 * 2 unfused exact, 3 fused tcgen05 bf16 (shape-specialised), 4 fused conv
 * front + exact dense, 5 generic tcgen05 bf16 layer chain (any dense model),
 * 6 fused exact with runtime dimensions (any small dense MLP), 7 conv front
 * (bf16 features) + tcgen05 bf16 dense chain (CNN at BF16) */
int smlrt_model_path(smlrt_model_t model, int32_t n_in_cols, int32_t* path);

/* gather_batch / concretize_to (bridge.py:388-395, 457-462): rows
 * [row_begin,row_end) of the plan -> dense [rows x n_cols] of out_dtype. */
int smlrt_gather(smlrt_plan_t plan, const void* const* array_ptrs,
                 const int32_t* array_dtypes, void* dense_out,
                 int32_t out_dtype, int64_t row_begin, int64_t row_end,
                 void* stream);

/* scatter_from (bridge.py:407-454): dense [rows x n_cols] -> arrays, with
 * the astype cast to each array's dtype.  FROM plans only. */
int smlrt_scatter(smlrt_plan_t plan, const void* dense_in, int32_t in_dtype,
                  void* const* array_ptrs, const int32_t* array_dtypes,
                  int64_t row_begin, int64_t row_end, void* stream);

/* models.infer (models.py:197-224) on a dense batch: x [rows x F] -> y
 * [rows x G].  Sets SMLRT_STATUS_NONFINITE in *d_status on NaN/inf. */
int smlrt_infer(smlrt_model_t model, const void* x, int32_t x_dtype,
                int64_t rows, void* y, int32_t y_dtype, void* stream,
                uint32_t* d_status);

/*
 * Runtime._run_surrogate (runtime.py:308-370) in one launch: gather through
 * `in_plan`, forward pass, scatter through `out_plan`, for sweep rows
 * [row_begin,row_end) (the multi-GPU shard range).  Validation errors are
 * returned before anything is launched; NonFinite via *d_status.
 * `workspace` (may be NULL for COMMIT_FUSED) must hold rows*G floats +
 * rows*max_width floats for the unfused path; smlrt_region_workspace()
 * reports the size.
 */
int smlrt_region_workspace(smlrt_plan_t in_plan, smlrt_plan_t out_plan,
                           smlrt_model_t model, int64_t rows, int32_t flags,
                           size_t* bytes);
int smlrt_region_infer(smlrt_plan_t in_plan, const void* const* in_ptrs,
                       const int32_t* in_dtypes, smlrt_plan_t out_plan,
                       void* const* out_ptrs, const int32_t* out_dtypes,
                       smlrt_model_t model, int64_t row_begin,
                       int64_t row_end, int32_t flags, void* workspace,
                       void* stream, uint32_t* d_status);

/*
 * Prepared region: the steady-state form of smlrt_region_infer for a
 * device-resident region invoked repeatedly with the same arrays, model and
 * rows (Runtime.invoke_region, runtime.py:227-277, once per application
 * step).  Arguments are validated and copied once; with use_graph the
 * launches are captured into a CUDA graph and every smlrt_region_run is one
 * graph launch, the stream synchronisation and the status check
 * (SMLRT_E_NONFINITE as smlrt_region_infer with SMLRT_SYNC_STATUS).
 * `d_status` is a device word used by the checked commit.  The plans, model
 * and arrays must outlive the handle.
 */
typedef struct smlrt_prepared_s* smlrt_prepared_t;
int smlrt_region_prepare(smlrt_plan_t in_plan, const void* const* in_ptrs,
                         const int32_t* in_dtypes, smlrt_plan_t out_plan,
                         void* const* out_ptrs, const int32_t* out_dtypes,
                         smlrt_model_t model, int64_t row_begin,
                         int64_t row_end, int32_t flags, uint32_t* d_status,
                         int32_t use_graph, smlrt_prepared_t* out);
int smlrt_region_run(smlrt_prepared_t prepared, void* stream);
/* the same, with the device time of the launches (CUDA events recorded on
 * `stream` around them) in *ms -- the bench's kernel-time measurement */
int smlrt_region_run_timed(smlrt_prepared_t prepared, void* stream, float* ms);
int smlrt_region_graphed(smlrt_prepared_t prepared, int32_t* graphed);
int smlrt_region_release(smlrt_prepared_t prepared);

/*
 * ml(collect) snapshot (runtime.py:279-306 feeding srdb.py:163-208): copy a
 * gathered dense tensor to pinned host memory on `side_stream`, ordered
 * after `after_event` (a cudaEvent_t recorded on the gather stream, may be
 * NULL); records a completion event the caller can wait on via
 * smlrt_collect_wait.
 */
int smlrt_collect_async(const void* dense_dev, size_t bytes, void* pinned_host,
                        void* side_stream, void* after_event);
int smlrt_collect_wait(void* side_stream);

/*
 * Host-path staging of a strided box (the e2e path of window functors, e.g.
 * C4's [k, 0:128, 0:128] = ([k, 16:144, 16:144])): copies the elements
 *   offset + z*slice + y*pitch + x,  x < width, y < height, z < depth
 * of `src` to the same element positions of `dst` (one cudaMemcpy3DAsync:
 * only the box's bytes cross PCIe).  direction: 0 host->device, 1
 * device->host.  slice must be a multiple of pitch.
 */
int smlrt_copy_box_async(void* dst, const void* src, int64_t elem_size, int64_t offset, int64_t width,
                         int64_t height, int64_t depth, int64_t pitch, int64_t slice, int32_t direction,
                         void* stream);

/* Diagnostic: one-CTA tcgen05 GEMM D[128 x N] = A[128 x K] * B[N x K]^T
 * (host f32 in, bf16 operands staged in the fused kernel's SW32/SW128
 * layouts, f32 out).  Validates descriptor encodings on a new device. */
int smlrt_tc_selftest(int K, int N, const float* A, const float* B, float* D);
/* Same with A staged in TMEM by tcgen05.st (the TS operand path). */
int smlrt_tc_selftest_ts(int K, int N, const float* A, const float* B, float* D);

/* Diagnostic: FP32 CUDA-core peak of the current device in flop/s for an
 * instruction mix: 0 = FFMA, 1 = FMUL + FADD (no contraction), 2 = packed
 * mul.rn.f32x2 + fma.rn.f32x2(p, 1, acc) -- the exact path's ordered
 * multiply-then-add on f32x2 pairs.  The bench's fp32 roofline denominator. */
int smlrt_fp32_peak(int32_t mode, double* flops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* SMLRT_B200_H */
