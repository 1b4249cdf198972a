// extern "C" entry points of libsmlrt_b200 (declared in include/smlrt_b200.h).
// Dispatch only: validation, device tables, and the choice of kernel.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

using namespace smlrt;

namespace {

int device_tables(smlrt_plan_t p, DevPlan* d, const int32_t* dtypes, int n) {
  int rc = p->tables(d);
  if (rc) return rc;
  d->all_f32 = 1;
  for (int i = 0; i < n; ++i) d->all_f32 &= dtypes[i] == SMLRT_F32;
  return SMLRT_OK;
}

// Keep up to kPoolKeep bytes of the device's stream-ordered pool across
// synchronisations, so per-call scratch is a pool hit after the first call;
// larger one-off scratch (e.g. a checked commit's staged output) goes back
// to the driver at the next synchronisation instead of staying reserved.
constexpr uint64_t kPoolKeep = 1ull << 30;
void warm_pool() {
  static int done_mask = 0;
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || (done_mask & (1 << d))) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
    uint64_t keep = kPoolKeep;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done_mask |= 1 << d;
}

struct Scratch {  // stream-ordered temporary
  void* p = nullptr;
  cudaStream_t s;
  explicit Scratch(cudaStream_t st) : s(st) { warm_pool(); }
  int alloc(size_t bytes) {
    if (bytes == 0) return SMLRT_OK;
    SMLRT_CUDA(cudaMallocAsync(&p, bytes, s));
    return SMLRT_OK;
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

int check_rows(smlrt_plan_t p, int64_t r0, int64_t r1) {
  if (r0 < 0 || r1 > p->n_rows || r0 > r1)
    return fail(SMLRT_E_INVALID, "row range [" + std::to_string(r0) + "," + std::to_string(r1) +
                                     ") outside the plan's " + std::to_string(p->n_rows) + " rows");
  return SMLRT_OK;
}

}  // namespace

smlrt_model_s::~smlrt_model_s() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  for (auto& L : layers) {
    cudaFree(L.w);
    cudaFree(L.b);
  }
  cudaFree(tc_blob);
  cudaFree(chain_blob);
  cudaFree(smm_blob);
  cudaFree(stc_blob);
  cudaSetDevice(prev);
}

extern "C" int smlrt_model_upload(const smlrt_layer_t* layers, int n_layers, int precision,
                                  int device, smlrt_model_t* out) {
  if (!layers || n_layers < 1 || !out) return fail(SMLRT_E_INVALID, "model_upload: no layers");
  if (precision != SMLRT_FP32_EXACT && precision != SMLRT_BF16)
    return fail(SMLRT_E_INVALID, "model_upload: unknown precision");
  for (int l = 0; l < n_layers; ++l) {
    const auto& L = layers[l];
    if (L.kind < SMLRT_DENSE || L.kind > SMLRT_MAXPOOL2D)
      return fail(SMLRT_E_INVALID, "model_upload: unknown layer kind");
    if (L.in < 1 || L.out < 1 || (L.kind != SMLRT_MAXPOOL2D && (!L.weights || !L.bias)))
      return fail(SMLRT_E_INVALID, "model_upload: empty layer " + std::to_string(l));
    if (L.activation < SMLRT_IDENTITY || L.activation > SMLRT_TANH)
      return fail(SMLRT_E_INVALID, "model_upload: unknown activation");
    if (l && L.in != layers[l - 1].out)
      return fail(SMLRT_E_MODEL_SHAPE, "model_upload: layer chain breaks at " + std::to_string(l));
    if (L.kind != SMLRT_DENSE) {
      const int k = L.kernel;
      if (k < 1 || L.stride != k || L.in_channels < 1 || L.in_h % k || L.in_w % k ||
          L.in != L.in_channels * L.in_h * L.in_w)
        return fail(SMLRT_E_MODEL_SHAPE, "model_upload: bad conv/pool geometry at layer " + std::to_string(l));
      if (L.out % ((L.in_h / k) * (L.in_w / k)))
        return fail(SMLRT_E_MODEL_SHAPE, "model_upload: bad conv/pool output width at layer " + std::to_string(l));
    }
  }
  int prev = 0;
  SMLRT_CUDA(cudaGetDevice(&prev));
  SMLRT_CUDA(cudaSetDevice(device));
  auto* m = new smlrt_model_s();
  m->precision = precision;
  m->device = device;
  m->n_layers = n_layers;
  m->in_features = layers[0].in;
  m->out_features = layers[n_layers - 1].out;
  m->max_width = 0;
  for (int l = 0; l < n_layers; ++l) {
    const auto& L = layers[l];
    DevLayer d;
    d.kind = L.kind;
    d.in = L.in;
    d.out = L.out;
    d.act = L.activation;
    d.kernel = L.kernel;
    d.stride = L.stride;
    d.in_c = L.in_channels;
    d.in_h = L.in_h;
    d.in_w = L.in_w;
    m->max_width = std::max(m->max_width, std::max(L.in, L.out));
    if (L.kind == SMLRT_MAXPOOL2D) {
      d.out_c = L.in_channels;
      m->layers.push_back(d);
      continue;
    }
    size_t nw, nb;
    if (L.kind == SMLRT_CONV2D) {
      d.out_c = L.out / ((L.in_h / L.kernel) * (L.in_w / L.kernel));
      nw = (size_t)d.out_c * L.in_channels * L.kernel * L.kernel;
      nb = (size_t)d.out_c;
    } else {
      nw = (size_t)L.in * L.out;
      nb = (size_t)L.out;
    }
    if (cudaMalloc(&d.w, nw * 4) != cudaSuccess || cudaMalloc(&d.b, nb * 4) != cudaSuccess ||
        cudaMemcpy(d.w, L.weights, nw * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d.b, L.bias, nb * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      m->layers.push_back(d);
      delete m;
      cudaSetDevice(prev);
      return fail(SMLRT_E_CUDA, "model_upload: device allocation/copy failed");
    }
    m->layers.push_back(d);
    m->host_params.insert(m->host_params.end(), L.weights, L.weights + nw);
    m->host_params.insert(m->host_params.end(), L.bias, L.bias + nb);
  }
  if (precision == SMLRT_BF16) {
    int rc = tc_pack_model(*m);
    if (rc) {
      std::string msg = smlrt_last_error();
      delete m;
      cudaSetDevice(prev);
      return fail(rc, msg);
    }
  }
  cudaSetDevice(prev);
  *out = m;
  return SMLRT_OK;
}

extern "C" int smlrt_model_free(smlrt_model_t m) {
  delete m;
  return SMLRT_OK;
}

extern "C" int smlrt_model_path(smlrt_model_t m, int32_t n_in_cols, int32_t* path) {
  if (!m || !path) return fail(SMLRT_E_INVALID, "model_path: null");
  (void)n_in_cols;
  DevPlan dummy{};
  *path = 2;
  if (cnn_model(*m)) {
    *path = m->precision == SMLRT_BF16 ? (m->chain_first > 0 ? 7 : 0) : 4;
  } else if (m->precision == SMLRT_BF16) {
    if (launch_region_tc(*m, dummy, nullptr, nullptr, 0, dummy, nullptr, nullptr, 0, 0, 0, nullptr,
                         0, nullptr, true) == SMLRT_OK)
      *path = 3;
    else
      *path = chain_ok(*m) ? 5 : 0;
  } else if (int k = exact_fused_kind(*m)) {
    *path = k;
  }
  return SMLRT_OK;
}

extern "C" int smlrt_gather(smlrt_plan_t p, const void* const* ptrs, const int32_t* dts, void* out,
                            int32_t out_dtype, int64_t r0, int64_t r1, void* stream) {
  if (!p || !ptrs || !dts || !out) return fail(SMLRT_E_INVALID, "gather: null argument");
  if (int rc = check_rows(p, r0, r1)) return rc;
  DevPlan d;
  if (int rc = device_tables(p, &d, dts, p->n_arrays)) return rc;
  return launch_gather(d, ptrs, dts, p->n_arrays, out, out_dtype, r0, r1, (cudaStream_t)stream);
}

extern "C" int smlrt_scatter(smlrt_plan_t p, const void* in, int32_t in_dtype, void* const* ptrs,
                             const int32_t* dts, int64_t r0, int64_t r1, void* stream) {
  if (!p || !ptrs || !dts || !in) return fail(SMLRT_E_INVALID, "scatter: null argument");
  if (p->direction != SMLRT_FROM) return fail(SMLRT_E_INVALID, "scatter needs a FROM plan");
  if (int rc = check_rows(p, r0, r1)) return rc;
  DevPlan d;
  if (int rc = device_tables(p, &d, dts, p->n_arrays)) return rc;
  return launch_scatter(d, in, in_dtype, ptrs, dts, p->n_arrays, r0, r1, (cudaStream_t)stream,
                        nullptr);
}

namespace {

// Layer-by-layer exact forward over dense f32 rows; ping-pong buffers.
int forward_unfused(const smlrt_model_s& m, const float* x, int64_t rows, float* y, float* t0,
                    float* t1, cudaStream_t s, uint32_t* status) {
  const float* cur = x;
  for (int l = 0; l < m.n_layers; ++l) {
    bool last = l == m.n_layers - 1;
    float* dst = last ? y : (l % 2 ? t1 : t0);
    if (int rc = launch_dense_exact_tiled(cur, rows, m.layers[l], dst, s, last ? status : nullptr)) return rc;
    cur = dst;
  }
  return SMLRT_OK;
}

constexpr int64_t kChunk = 1 << 16;  // rows per unfused chunk (bounds scratch)

}  // namespace

extern "C" int smlrt_infer(smlrt_model_t m, const void* x, int32_t x_dtype, int64_t rows, void* y,
                           int32_t y_dtype, void* stream, uint32_t* status) {
  if (!m || !x || !y || !status) return fail(SMLRT_E_INVALID, "infer: null argument");
  if (rows <= 0) return SMLRT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t ch = std::min(rows, cnn_model(*m) ? (int64_t)4096 : kChunk);
  Scratch sc(s);
  size_t per = (size_t)m->in_features + 2 * (size_t)m->max_width + m->out_features;
  if (int rc = sc.alloc(per * ch * 4)) return rc;
  float* xin = (float*)sc.p;
  float* t0 = xin + ch * m->in_features;
  float* t1 = t0 + ch * m->max_width;
  float* yo = t1 + ch * m->max_width;
  size_t xs = x_dtype == SMLRT_F32 ? 4 : 8, ys = y_dtype == SMLRT_F32 ? 4 : 8;
  for (int64_t r = 0; r < rows; r += ch) {
    int64_t n = std::min(ch, rows - r);
    const char* xp = (const char*)x + r * m->in_features * xs;
    if (int rc = launch_convert(xp, x_dtype, xin, SMLRT_F32, n * m->in_features, s)) return rc;
    if (cnn_model(*m)) {
      if (int rc = infer_cnn_dense(*m, xin, n, yo, s, status)) return rc;
    } else if (int rc = forward_unfused(*m, xin, n, yo, t0, t1, s, status)) {
      return rc;
    }
    char* yp = (char*)y + r * m->out_features * ys;
    if (int rc = launch_convert(yo, SMLRT_F32, yp, y_dtype, n * m->out_features, s)) return rc;
  }
  return SMLRT_OK;
}

extern "C" int smlrt_region_workspace(smlrt_plan_t in, smlrt_plan_t out, smlrt_model_t m, int64_t rows,
                                      int32_t flags, size_t* bytes) {
  if (!in || !out || !m || !bytes) return fail(SMLRT_E_INVALID, "region_workspace: null");
  size_t b = 0;
  if (flags & SMLRT_COMMIT_CHECKED) b += (size_t)rows * m->out_features * 4;
  *bytes = b;
  return SMLRT_OK;
}

static int region_launch(smlrt_plan_t pin, const void* const* in_ptrs, const int32_t* in_dt, smlrt_plan_t pout,
                         void* const* out_ptrs, const int32_t* out_dt, smlrt_model_t m, int64_t r0, int64_t r1,
                         int32_t flags, void* workspace, cudaStream_t s, uint32_t* status);

extern "C" int smlrt_region_infer(smlrt_plan_t pin, const void* const* in_ptrs, const int32_t* in_dt,
                                  smlrt_plan_t pout, void* const* out_ptrs, const int32_t* out_dt,
                                  smlrt_model_t m, int64_t r0, int64_t r1, int32_t flags,
                                  void* workspace, void* stream, uint32_t* status) {
  if (!pin || !pout || !m || !in_ptrs || !out_ptrs || !in_dt || !out_dt || !status)
    return fail(SMLRT_E_INVALID, "region_infer: null argument");
  if (pin->direction != SMLRT_TO || pout->direction != SMLRT_FROM)
    return fail(SMLRT_E_INVALID, "region_infer: plans have the wrong directions");
  // runtime.py:327-338
  if (pin->n_cols != m->in_features)
    return fail(SMLRT_E_MODEL_SHAPE, "region gathers " + std::to_string(pin->n_cols) +
                                         " features, model expects " + std::to_string(m->in_features));
  if (pout->n_cols != m->out_features)
    return fail(SMLRT_E_MODEL_SHAPE, "region scatters " + std::to_string(pout->n_cols) +
                                         " features, model emits " + std::to_string(m->out_features));
  if (pout->n_rows != pin->n_rows)
    return fail(SMLRT_E_MODEL_SHAPE, "output map sweeps " + std::to_string(pout->n_rows) +
                                         " entries, batch holds " + std::to_string(pin->n_rows));
  if (int rc = check_rows(pin, r0, r1)) return rc;
  if (r1 == r0) return SMLRT_OK;
  int dev = 0;
  SMLRT_CUDA(cudaGetDevice(&dev));
  if (dev != m->device) return fail(SMLRT_E_INVALID, "region_infer: model lives on another device");
  cudaStream_t s = (cudaStream_t)stream;
  if (flags & SMLRT_SYNC_STATUS) {
    if (!(flags & SMLRT_COMMIT_CHECKED)) {
      // zero-copy status: a mapped pinned word the kernels store into, reset
      // by the host -- launch + sync only, no memset or read-back copy
      static thread_local volatile uint32_t* h_flag = nullptr;  // one per host thread
      if (!h_flag) {
        void* p = nullptr;
        SMLRT_CUDA(cudaHostAlloc(&p, sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable));
        h_flag = static_cast<volatile uint32_t*>(p);
      }
      uint32_t* d_flag = nullptr;
      SMLRT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_flag), const_cast<uint32_t*>(h_flag), 0));
      *h_flag = 0u;
      const int rc = region_launch(pin, in_ptrs, in_dt, pout, out_ptrs, out_dt, m, r0, r1, flags, workspace, s, d_flag);
      if (rc) return rc;
      SMLRT_CUDA(cudaStreamSynchronize(s));
      if (*h_flag & SMLRT_STATUS_NONFINITE) return fail(SMLRT_E_NONFINITE, "forward pass produced NaN/inf");
      return SMLRT_OK;
    }
    // checked commit: the gated scatter reads the status word, keep it in HBM
    SMLRT_CUDA(cudaMemsetAsync(status, 0, sizeof(uint32_t), s));
    const int rc = region_launch(pin, in_ptrs, in_dt, pout, out_ptrs, out_dt, m, r0, r1, flags, workspace, s, status);
    if (rc) return rc;
    static thread_local uint32_t* h_status = nullptr;  // pinned, one per host thread
    if (!h_status) SMLRT_CUDA(cudaMallocHost(&h_status, sizeof(uint32_t)));
    SMLRT_CUDA(cudaMemcpyAsync(h_status, status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SMLRT_CUDA(cudaStreamSynchronize(s));
    if (*h_status & SMLRT_STATUS_NONFINITE) return fail(SMLRT_E_NONFINITE, "forward pass produced NaN/inf");
    return SMLRT_OK;
  }
  return region_launch(pin, in_ptrs, in_dt, pout, out_ptrs, out_dt, m, r0, r1, flags, workspace, s, status);
}

// the launches of smlrt_region_infer (validated arguments)
static int region_launch(smlrt_plan_t pin, const void* const* in_ptrs, const int32_t* in_dt, smlrt_plan_t pout,
                         void* const* out_ptrs, const int32_t* out_dt, smlrt_model_t m, int64_t r0, int64_t r1,
                         int32_t flags, void* workspace, cudaStream_t s, uint32_t* status) {
  DevPlan din, dout;
  if (int rc = device_tables(pin, &din, in_dt, pin->n_arrays)) return rc;
  if (int rc = device_tables(pout, &dout, out_dt, pout->n_arrays)) return rc;
  int64_t rows = r1 - r0;
  bool checked = flags & SMLRT_COMMIT_CHECKED;
  Scratch stage_sc(s);
  float* staged = nullptr;
  if (checked) {
    if (workspace) {
      staged = (float*)workspace;
    } else {
      if (int rc = stage_sc.alloc((size_t)rows * m->out_features * 4)) return rc;
      staged = (float*)stage_sc.p;
    }
  }
  int rc = SMLRT_E_UNSUPPORTED;
  if (cnn_model(*m)) {
    warm_pool();
    if (int e = launch_region_cnn(*m, din, in_ptrs, in_dt, pin->n_arrays, dout, out_ptrs, out_dt, pout->n_arrays,
                                  r0, r1, staged, s, status))
      return e;
    rc = SMLRT_OK;
  } else if (!(flags & SMLRT_FORCE_UNFUSED)) {
    if (m->precision == SMLRT_BF16)
      rc = launch_region_tc(*m, din, in_ptrs, in_dt, pin->n_arrays, dout, out_ptrs, out_dt,
                            pout->n_arrays, r0, r1, staged, s, status, false);
    else {
      // the halo-stencil shape (C5): TMA-fed exact kernel; SMLRT_STENCIL_EXACT=0 (A/B) skips it
      static const bool sx_on = [] {
        const char* e = std::getenv("SMLRT_STENCIL_EXACT");
        return !(e && e[0] == '0');
      }();
      if (sx_on)
        rc = launch_region_stencil_exact(*m, din, in_ptrs, in_dt, dout, out_ptrs, out_dt, r0, r1, staged, s, status);
      if (rc == SMLRT_E_UNSUPPORTED)
        rc = launch_region_exact_fused(*m, din, in_ptrs, in_dt, pin->n_arrays, dout, out_ptrs, out_dt,
                                       pout->n_arrays, r0, r1, staged, s, status, false);
    }
    if (rc != SMLRT_OK && rc != SMLRT_E_UNSUPPORTED) return rc;
    if (rc == SMLRT_E_UNSUPPORTED && m->precision == SMLRT_BF16)
      return rc;  // launch_region_chain's message: the model has non-dense or > 4096-wide layers
  }
  if (rc == SMLRT_E_UNSUPPORTED) {
    // unfused exact path: gather -> per-layer kernels -> scatter, chunked
    int64_t ch = std::min(rows, kChunk);
    Scratch sc(s);
    size_t per = (size_t)m->in_features + 2 * (size_t)m->max_width + m->out_features;
    if (int e = sc.alloc(per * ch * 4)) return e;
    float* xin = (float*)sc.p;
    float* t0 = xin + ch * m->in_features;
    float* t1 = t0 + ch * m->max_width;
    float* yo = t1 + ch * m->max_width;
    for (int64_t r = r0; r < r1; r += ch) {
      int64_t n = std::min(ch, r1 - r);
      if (int e = launch_gather(din, in_ptrs, in_dt, pin->n_arrays, xin, SMLRT_F32, r, r + n, s)) return e;
      float* ydst = checked ? staged + (r - r0) * m->out_features : yo;
      if (int e = forward_unfused(*m, xin, n, ydst, t0, t1, s, status)) return e;
      if (!checked)
        if (int e = launch_scatter(dout, ydst, SMLRT_F32, out_ptrs, out_dt, pout->n_arrays, r, r + n, s,
                                   nullptr))
          return e;
    }
  }
  if (checked) {
    // commit: a no-op on device when the status word is non-zero
    if (int e = launch_scatter(dout, staged, SMLRT_F32, out_ptrs, out_dt, pout->n_arrays, r0, r1, s,
                               status))
      return e;
  }
  return SMLRT_OK;
}

// ---------------------------------------------------------------- prepared regions
// A device-resident region invoked again and again with the same arrays,
// model and row range (the reference's steady state: one invoke_region per
// application timestep, runtime.py:227-277): validated once, its launches
// (scratch allocation, gather/forward/scatter kernels, tensor maps baked into
// kernel parameters) captured once into a CUDA graph, then replayed -- one
// cudaGraphLaunch per call instead of the per-launch host work (tables,
// tensor-map encoding, scratch allocation) that otherwise sits between the
// caller's stream work and the first kernel.  Capture failures fall back to
// the direct launches (same kernels).
struct smlrt_prepared_s {
  smlrt_plan_t pin = nullptr, pout = nullptr;
  smlrt_model_t m = nullptr;
  std::vector<const void*> in_ptrs;
  std::vector<void*> out_ptrs;
  std::vector<int32_t> in_dt, out_dt;
  int64_t r0 = 0, r1 = 0;
  int32_t flags = 0;
  uint32_t* status = nullptr;        // checked commit: device status word
  volatile uint32_t* h_flag = nullptr;  // fused commit: mapped pinned flag
  uint32_t* d_flag = nullptr;
  uint32_t* h_status = nullptr;      // checked commit: pinned read-back
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  unsigned long long kernels = 0;    // kernel nodes per replay (launch counter)
  cudaEvent_t ev[2] = {nullptr, nullptr};  // smlrt_region_run_timed
  ~smlrt_prepared_s() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (h_flag) cudaFreeHost(const_cast<uint32_t*>(h_flag));
    if (h_status) cudaFreeHost(h_status);
  }
};

namespace {
// the launches of one prepared call on stream s (no host sync)
int prepared_enqueue(smlrt_prepared_s& p, cudaStream_t s) {
  const bool checked = p.flags & SMLRT_COMMIT_CHECKED;
  uint32_t* st = checked ? p.status : p.d_flag;
  if (checked) SMLRT_CUDA(cudaMemsetAsync(p.status, 0, sizeof(uint32_t), s));
  if (int rc = region_launch(p.pin, p.in_ptrs.data(), p.in_dt.data(), p.pout, p.out_ptrs.data(), p.out_dt.data(),
                             p.m, p.r0, p.r1, p.flags & ~SMLRT_SYNC_STATUS, nullptr, s, st))
    return rc;
  if (checked) SMLRT_CUDA(cudaMemcpyAsync(p.h_status, p.status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  return SMLRT_OK;
}
}  // namespace

extern "C" int smlrt_region_prepare(smlrt_plan_t pin, const void* const* in_ptrs, const int32_t* in_dt,
                                    smlrt_plan_t pout, void* const* out_ptrs, const int32_t* out_dt,
                                    smlrt_model_t m, int64_t r0, int64_t r1, int32_t flags, uint32_t* d_status,
                                    int32_t use_graph, smlrt_prepared_t* out) {
  if (!pin || !pout || !m || !in_ptrs || !out_ptrs || !in_dt || !out_dt || !d_status || !out)
    return fail(SMLRT_E_INVALID, "region_prepare: null argument");
  if (pin->direction != SMLRT_TO || pout->direction != SMLRT_FROM)
    return fail(SMLRT_E_INVALID, "region_prepare: plans have the wrong directions");
  if (pin->n_cols != m->in_features || pout->n_cols != m->out_features || pout->n_rows != pin->n_rows)
    return fail(SMLRT_E_MODEL_SHAPE, "region_prepare: plans and model disagree (run smlrt_region_infer first)");
  if (int rc = check_rows(pin, r0, r1)) return rc;
  int dev = 0;
  SMLRT_CUDA(cudaGetDevice(&dev));
  if (dev != m->device) return fail(SMLRT_E_INVALID, "region_prepare: model lives on another device");
  auto* p = new smlrt_prepared_s();
  p->pin = pin;
  p->pout = pout;
  p->m = m;
  p->in_ptrs.assign(in_ptrs, in_ptrs + pin->n_arrays);
  p->out_ptrs.assign(out_ptrs, out_ptrs + pout->n_arrays);
  p->in_dt.assign(in_dt, in_dt + pin->n_arrays);
  p->out_dt.assign(out_dt, out_dt + pout->n_arrays);
  p->r0 = r0;
  p->r1 = r1;
  p->flags = flags | SMLRT_SYNC_STATUS;
  p->status = d_status;
  auto bail = [&](int rc) {
    std::string msg = smlrt_last_error();
    delete p;
    return fail(rc, msg);
  };
  void* hp = nullptr;
  if (cudaHostAlloc(&hp, sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&p->h_status), sizeof(uint32_t), cudaHostAllocPortable) != cudaSuccess)
    return bail(fail(SMLRT_E_CUDA, "region_prepare: pinned status allocation failed"));
  p->h_flag = static_cast<volatile uint32_t*>(hp);
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->d_flag), hp, 0) != cudaSuccess)
    return bail(fail(SMLRT_E_CUDA, "region_prepare: mapped status pointer"));
  if (r1 > r0 && use_graph) {
    // device tables and the pool setting outside the capture (their first
    // use allocates, copies or sets pool attributes: not capturable)
    warm_pool();
    DevPlan d;
    if (int rc = device_tables(pin, &d, in_dt, pin->n_arrays)) return bail(rc);
    if (int rc = device_tables(pout, &d, out_dt, pout->n_arrays)) return bail(rc);
    cudaStream_t cs = nullptr;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess) {
      const unsigned long long n0 = smlrt_launch_count();
      bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      const int rc = ok ? prepared_enqueue(*p, cs) : SMLRT_E_CUDA;
      cudaGraph_t g = nullptr;
      const bool ended = ok && cudaStreamEndCapture(cs, &g) == cudaSuccess && g != nullptr;
      if (rc == SMLRT_OK && ended && cudaGraphInstantiate(&p->exec, g, 0) == cudaSuccess) {
        p->graph = g;
        p->kernels = smlrt_launch_count() - n0;
        g_launches.fetch_sub(p->kernels, std::memory_order_relaxed);  // captured, not launched
      } else {
        if (g) cudaGraphDestroy(g);
        p->exec = nullptr;
        g_launches.fetch_sub(smlrt_launch_count() - n0, std::memory_order_relaxed);
      }
      cudaGetLastError();  // a refused capture leaves a sticky-free error code behind
      cudaStreamDestroy(cs);
    }
  }
  *out = p;
  return SMLRT_OK;
}

namespace {
int prepared_run(smlrt_prepared_t p, cudaStream_t s, float* ms) {
  if (!p) return fail(SMLRT_E_INVALID, "region_run: null handle");
  if (p->r1 == p->r0) {
    if (ms) *ms = 0.0f;
    return SMLRT_OK;
  }
  const bool checked = p->flags & SMLRT_COMMIT_CHECKED;
  *p->h_flag = 0u;
  if (ms) {
    for (auto& e : p->ev)
      if (!e) SMLRT_CUDA(cudaEventCreate(&e));
    SMLRT_CUDA(cudaEventRecord(p->ev[0], s));
  }
  if (p->exec) {
    SMLRT_CUDA(cudaGraphLaunch(p->exec, s));
    g_launches.fetch_add(p->kernels, std::memory_order_relaxed);
  } else if (int rc = prepared_enqueue(*p, s)) {
    return rc;
  }
  if (ms) SMLRT_CUDA(cudaEventRecord(p->ev[1], s));
  SMLRT_CUDA(cudaStreamSynchronize(s));
  if (ms) SMLRT_CUDA(cudaEventElapsedTime(ms, p->ev[0], p->ev[1]));
  const uint32_t st = checked ? *p->h_status : *p->h_flag;
  if (st & SMLRT_STATUS_NONFINITE) return fail(SMLRT_E_NONFINITE, "forward pass produced NaN/inf");
  return SMLRT_OK;
}
}  // namespace

extern "C" int smlrt_region_run(smlrt_prepared_t p, void* stream) {
  return prepared_run(p, (cudaStream_t)stream, nullptr);
}

extern "C" int smlrt_region_run_timed(smlrt_prepared_t p, void* stream, float* ms) {
  if (!ms) return fail(SMLRT_E_INVALID, "region_run_timed: null ms");
  return prepared_run(p, (cudaStream_t)stream, ms);
}

extern "C" int smlrt_region_graphed(smlrt_prepared_t p, int32_t* graphed) {
  if (!p || !graphed) return fail(SMLRT_E_INVALID, "region_graphed: null argument");
  *graphed = p->exec != nullptr;
  return SMLRT_OK;
}

extern "C" int smlrt_region_release(smlrt_prepared_t p) {
  delete p;
  return SMLRT_OK;
}

extern "C" int smlrt_collect_async(const void* dense_dev, size_t bytes, void* pinned_host,
                                   void* side_stream, void* after_event) {
  if (!dense_dev || !pinned_host) return fail(SMLRT_E_INVALID, "collect_async: null argument");
  cudaStream_t s = (cudaStream_t)side_stream;
  if (after_event) SMLRT_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)after_event, 0));
  SMLRT_CUDA(cudaMemcpyAsync(pinned_host, dense_dev, bytes, cudaMemcpyDeviceToHost, s));
  return SMLRT_OK;
}

extern "C" int smlrt_copy_box_async(void* dst, const void* src, int64_t esz, int64_t offset, int64_t width,
                                    int64_t height, int64_t depth, int64_t pitch, int64_t slice, int32_t direction,
                                    void* stream) {
  if (!dst || !src) return fail(SMLRT_E_INVALID, "copy_box: null pointer");
  if (esz <= 0 || width <= 0 || height <= 0 || depth <= 0 || pitch < width || slice < pitch * height ||
      slice % pitch != 0 || offset < 0)
    return fail(SMLRT_E_INVALID, "copy_box: inconsistent box geometry");
  const int64_t z0 = offset / slice, rem = offset % slice, y0 = rem / pitch, x0 = rem % pitch;
  if (x0 + width > pitch) return fail(SMLRT_E_INVALID, "copy_box: box rows wrap the pitch");
  cudaMemcpy3DParms p{};
  p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), (size_t)(pitch * esz), (size_t)pitch, (size_t)(slice / pitch));
  p.dstPtr = make_cudaPitchedPtr(dst, (size_t)(pitch * esz), (size_t)pitch, (size_t)(slice / pitch));
  p.srcPos = make_cudaPos((size_t)(x0 * esz), (size_t)y0, (size_t)z0);
  p.dstPos = p.srcPos;
  p.extent = make_cudaExtent((size_t)(width * esz), (size_t)height, (size_t)depth);
  p.kind = direction == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  SMLRT_CUDA(cudaMemcpy3DAsync(&p, (cudaStream_t)stream));
  return SMLRT_OK;
}

extern "C" int smlrt_collect_wait(void* side_stream) {
  SMLRT_CUDA(cudaStreamSynchronize((cudaStream_t)side_stream));
  return SMLRT_OK;
}
