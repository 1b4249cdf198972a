// Plan compiler: flattens wrap_tensors' views into a per-column address table,
// validates flat bounds, proves scatter injectivity once, uploads lazily.
//
// Reference behaviour it replaces:
//   bridge.py:288-344   wrap_tensors (views, eager bounds)
//   bridge.py:351-381   compose_tensor (column order: views in RHS order,
//                       feature axes row-major)
//   bridge.py:437-448   scatter_from injectivity (np.unique over all
//                       destination addresses, every call)  -> here once.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "common.cuh"

namespace {

thread_local std::string g_err;

// Mixed-radix proof that {sum_k i_k * s_k : 0 <= i_k < n_k} has no repeats:
// sorted by stride, each stride must exceed the span of all smaller ones.
bool lattice_injective(int n, const int64_t* extent, const int64_t* stride, int64_t* span) {
  std::vector<std::pair<int64_t, int64_t>> d;
  for (int k = 0; k < n; ++k)
    if (extent[k] > 1) d.push_back({stride[k], extent[k]});
  std::sort(d.begin(), d.end());
  int64_t reach = 0;  // largest offset reachable with the smaller strides
  for (auto& [s, e] : d) {
    if (s <= reach || s == 0) return false;
    reach += s * (e - 1);
  }
  *span = reach;
  return true;
}

}  // namespace

namespace smlrt {
void set_error(const std::string& m) { g_err = m; }
int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}
}  // namespace smlrt

using namespace smlrt;

extern "C" const char* smlrt_last_error(void) { return g_err.c_str(); }
extern "C" const char* smlrt_version(void) { return "smlrt_b200 0.1.0 (sm_100a)"; }

namespace smlrt {
std::atomic<unsigned long long> g_launches{0};
}
extern "C" unsigned long long smlrt_launch_count(void) { return smlrt::g_launches.load(); }

smlrt_plan_s::~smlrt_plan_s() {
  int prev = 0;
  cudaGetDevice(&prev);
  for (auto& [d, t] : dev) {
    cudaSetDevice(d);
    cudaFree(t.col_off);
    cudaFree(t.col_arr);
    cudaFree(t.col_str);
  }
  cudaSetDevice(prev);
}

int smlrt_plan_s::tables(DevPlan* p) {
  int d = 0;
  SMLRT_CUDA(cudaGetDevice(&d));
  std::lock_guard<std::mutex> lk(mu);
  auto it = dev.find(d);
  if (it == dev.end()) {
    DeviceTables t;
    size_t nc = (size_t)n_cols;
    SMLRT_CUDA(cudaMalloc(&t.col_off, nc * sizeof(int64_t)));
    SMLRT_CUDA(cudaMalloc(&t.col_arr, nc * sizeof(int32_t)));
    SMLRT_CUDA(cudaMalloc(&t.col_str, std::max<size_t>(1, nc * n_sweep) * sizeof(int64_t)));
    SMLRT_CUDA(cudaMemcpy(t.col_off, col_off.data(), nc * sizeof(int64_t), cudaMemcpyHostToDevice));
    SMLRT_CUDA(cudaMemcpy(t.col_arr, col_arr.data(), nc * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (!col_str.empty())
      SMLRT_CUDA(cudaMemcpy(t.col_str, col_str.data(), col_str.size() * sizeof(int64_t),
                            cudaMemcpyHostToDevice));
    it = dev.emplace(d, t).first;
  }
  memset(p, 0, sizeof(*p));
  p->n_sweep = n_sweep;
  p->n_cols = n_cols;
  p->uniform = uniform;
  p->n_rows = n_rows;
  p->uarray = uarray;
  for (int k = 0; k < SMLRT_MAX_SWEEP; ++k) {
    p->ustride[k] = ustride[k];
    p->sdiv[k] = FastDiv(k < n_sweep ? (uint32_t)sweep[k] : 1u);
  }
  p->cdiv = FastDiv((uint32_t)n_cols);
  p->dense_rows = dense_rows;
  p->col_off0 = col_off.empty() ? 0 : col_off[0];
  p->win_w = win_w;
  p->win_pitch = win_pitch;
  p->uarray_numel = uniform && uarray < (int)array_numel.size() ? array_numel[uarray] : 0;
  for (int c = 0; c < n_cols && c < SMLRT_INLINE_COLS; ++c) p->col_inl[c] = col_off[c];
  p->col_off = it->second.col_off;
  p->col_arr = it->second.col_arr;
  p->col_str = it->second.col_str;
  return SMLRT_OK;
}

extern "C" int smlrt_plan_create(const smlrt_view_t* views, int n_views, int n_sweep,
                                 const int64_t* sweep_shape, int direction,
                                 const int64_t* array_numel, int n_arrays, smlrt_plan_t* out) {
  if (!views || n_views < 1 || !out || !array_numel || n_arrays < 1)
    return fail(SMLRT_E_INVALID, "plan_create: empty view list or null argument");
  if (n_sweep < 1 || n_sweep > SMLRT_MAX_SWEEP)
    return fail(SMLRT_E_ARITY, "plan_create: sweep rank " + std::to_string(n_sweep) +
                                   " outside 1.." + std::to_string(SMLRT_MAX_SWEEP));
  if (direction != SMLRT_TO && direction != SMLRT_FROM)
    return fail(SMLRT_E_INVALID, "plan_create: bad direction");
  auto* p = new smlrt_plan_s();
  p->direction = direction;
  p->n_sweep = n_sweep;
  p->n_arrays = n_arrays;
  p->n_rows = 1;
  for (int k = 0; k < n_sweep; ++k) {
    if (sweep_shape[k] < 1) {
      delete p;
      return fail(SMLRT_E_SHAPE, "plan_create: empty sweep extent");
    }
    p->sweep[k] = sweep_shape[k];
    p->n_rows *= sweep_shape[k];
  }
  if (p->n_rows >= (1ll << 32)) {
    delete p;
    return fail(SMLRT_E_UNSUPPORTED, "plan_create: more than 2^32 sweep rows per plan; shard it");
  }
  p->views.assign(views, views + n_views);
  p->array_numel.assign(array_numel, array_numel + n_arrays);

  // ---- bounds (flat) and column table ----
  for (int v = 0; v < n_views; ++v) {
    const smlrt_view_t& w = views[v];
    if (w.array < 0 || w.array >= n_arrays || w.n_feat < 1 || w.n_feat > SMLRT_MAX_FEAT) {
      delete p;
      return fail(SMLRT_E_INVALID, "plan_create: bad view " + std::to_string(v));
    }
    int64_t lo = w.base, hi = w.base;
    for (int k = 0; k < n_sweep; ++k) {
      int64_t e = (p->sweep[k] - 1) * w.sweep_stride[k];
      (e < 0 ? lo : hi) += e;
    }
    int64_t ncol = 1;
    for (int a = 0; a < w.n_feat; ++a) {
      if (w.feat_count[a] < 1) {
        delete p;
        return fail(SMLRT_E_SHAPE, "plan_create: empty feature axis");
      }
      int64_t e = (w.feat_count[a] - 1) * w.feat_stride[a];
      (e < 0 ? lo : hi) += e;
      ncol *= w.feat_count[a];
    }
    if (lo < 0 || hi >= array_numel[w.array]) {
      delete p;
      return fail(SMLRT_E_OOB, "view " + std::to_string(v) + " addresses elements " +
                                   std::to_string(lo) + ".." + std::to_string(hi) +
                                   " of a storage holding " + std::to_string(array_numel[w.array]));
    }
    if (direction == SMLRT_FROM && ncol != 1) {
      delete p;
      return fail(SMLRT_E_NONINJECTIVE,
                  "scatter view with a feature range gives elements several destinations");
    }
    // row-major enumeration of the feature axes
    std::vector<int64_t> idx(w.n_feat, 0);
    for (int64_t c = 0; c < ncol; ++c) {
      int64_t off = w.base;
      for (int a = 0; a < w.n_feat; ++a) off += idx[a] * w.feat_stride[a];
      p->col_off.push_back(off);
      p->col_arr.push_back(w.array);
      for (int k = 0; k < n_sweep; ++k) p->col_str.push_back(w.sweep_stride[k]);
      for (int a = w.n_feat - 1; a >= 0; --a) {
        if (++idx[a] < w.feat_count[a]) break;
        idx[a] = 0;
      }
    }
  }
  if (p->col_off.size() >= (1u << 31)) {
    delete p;
    return fail(SMLRT_E_UNSUPPORTED, "plan_create: too many columns");
  }
  p->n_cols = (int)p->col_off.size();

  // ---- uniformity / dense rows ----
  p->uniform = true;
  p->uarray = views[0].array;
  for (int k = 0; k < n_sweep; ++k) p->ustride[k] = views[0].sweep_stride[k];
  for (int v = 1; v < n_views; ++v) {
    if (views[v].array != p->uarray) p->uniform = false;
    for (int k = 0; k < n_sweep; ++k)
      if (views[v].sweep_stride[k] != p->ustride[k]) p->uniform = false;
  }
  if (p->uniform) {
    bool run = true;
    for (int c = 1; c < p->n_cols; ++c)
      if (p->col_off[c] != p->col_off[0] + c) run = false;
    p->dense_rows = run && n_sweep == 1;
    p->row_pitch = p->dense_rows ? p->ustride[0] : 0;
  }

  // ---- 2-D window detection (one view, two feature axes, inner stride 1) ----
  if (p->uniform && n_views == 1 && views[0].n_feat == 2 && views[0].feat_stride[1] == 1) {
    p->win_w = (int)views[0].feat_count[1];
    p->win_pitch = views[0].feat_stride[0];
  }

  // ---- injectivity (FROM) ----
  if (direction == SMLRT_FROM) {
    bool proven = false;
    if (p->uniform) {
      int64_t span = 0;
      if (lattice_injective(n_sweep, p->sweep, p->ustride, &span)) {
        std::vector<int64_t> b(p->col_off);
        std::sort(b.begin(), b.end());
        proven = true;
        for (size_t i = 1; i < b.size(); ++i)
          if (b[i] - b[i - 1] <= span) proven = false;
      }
      // otherwise inconclusive (e.g. strides (2,3) over (3,2) are injective
      // without being mixed-radix): fall through to the exact bitmap
    }
    if (!proven) {
      // exact check: bitmap over each destination array's touched span
      for (int a = 0; a < n_arrays; ++a) {
        int64_t lo = INT64_MAX, hi = -1;
        for (int v = 0; v < n_views; ++v) {
          if (views[v].array != a) continue;
          int64_t l = views[v].base, h = views[v].base;
          for (int k = 0; k < n_sweep; ++k) h += (p->sweep[k] - 1) * views[v].sweep_stride[k];
          lo = std::min(lo, l);
          hi = std::max(hi, h);
        }
        if (hi < 0) continue;
        if (hi - lo + 1 > (1ll << 34)) {
          delete p;
          return fail(SMLRT_E_UNSUPPORTED, "injectivity check span too large");
        }
        std::vector<uint64_t> bits((size_t)((hi - lo) / 64 + 1), 0);
        std::vector<int64_t> idx(n_sweep);
        for (int v = 0; v < n_views; ++v) {
          const smlrt_view_t& w = views[v];
          if (w.array != a) continue;
          std::fill(idx.begin(), idx.end(), 0);
          for (int64_t r = 0; r < p->n_rows; ++r) {
            int64_t addr = w.base - lo;
            for (int k = 0; k < n_sweep; ++k) addr += idx[k] * w.sweep_stride[k];
            uint64_t m = 1ull << (addr & 63);
            if (bits[addr >> 6] & m) {
              delete p;
              return fail(SMLRT_E_NONINJECTIVE,
                          "scatter maps two tensor elements onto array element " +
                              std::to_string(addr + lo));
            }
            bits[addr >> 6] |= m;
            for (int k = n_sweep - 1; k >= 0; --k) {
              if (++idx[k] < p->sweep[k]) break;
              idx[k] = 0;
            }
          }
        }
      }
    }
    p->injective = true;
  }
  *out = p;
  return SMLRT_OK;
}

extern "C" int smlrt_plan_info(smlrt_plan_t p, smlrt_plan_info_t* info) {
  if (!p || !info) return fail(SMLRT_E_INVALID, "plan_info: null");
  info->n_rows = p->n_rows;
  info->n_cols = p->n_cols;
  info->n_views = (int32_t)p->views.size();
  info->n_arrays = p->n_arrays;
  info->uniform = p->uniform;
  info->dense_rows = p->dense_rows;
  info->injective = p->injective;
  info->row_pitch = p->row_pitch;
  return SMLRT_OK;
}

extern "C" int smlrt_plan_row_ranges(smlrt_plan_t p, int64_t r0, int64_t r1, int64_t* ranges, int32_t max_ranges,
                                     int32_t* n_ranges, int32_t* exact) {
  if (!p || !ranges || !n_ranges || !exact) return fail(SMLRT_E_INVALID, "plan_row_ranges: null");
  if (!p->uniform || p->n_sweep != 1) return fail(SMLRT_E_UNSUPPORTED, "plan_row_ranges: needs a uniform 1-D plan");
  if (r0 < 0 || r1 > p->n_rows || r0 >= r1) return fail(SMLRT_E_INVALID, "plan_row_ranges: bad row range");
  const int64_t s = p->ustride[0];
  if (s < 1) return fail(SMLRT_E_UNSUPPORTED, "plan_row_ranges: non-positive row stride");
  std::vector<std::pair<int64_t, int64_t>> iv;
  iv.reserve(p->n_cols);
  for (int c = 0; c < p->n_cols; ++c) iv.push_back({p->col_off[c] + r0 * s, p->col_off[c] + (r1 - 1) * s + 1});
  std::sort(iv.begin(), iv.end());
  int n = 0;
  for (const auto& v : iv) {
    if (n > 0 && v.first <= ranges[2 * n - 1]) {
      ranges[2 * n - 1] = std::max(ranges[2 * n - 1], v.second);
      continue;
    }
    if (n == max_ranges) return fail(SMLRT_E_UNSUPPORTED, "plan_row_ranges: more ranges than max_ranges");
    ranges[2 * n] = v.first;
    ranges[2 * n + 1] = v.second;
    ++n;
  }
  *n_ranges = n;
  *exact = (s == 1 || (p->dense_rows && s == p->n_cols)) ? 1 : 0;
  return SMLRT_OK;
}

extern "C" int smlrt_plan_destroy(smlrt_plan_t p) {
  delete p;
  return SMLRT_OK;
}
