// api.cu -- the C ABI of libcorr.so (include/corr.h): validation, field handles,
// stream plumbing and dispatch to the hot-path kernels.  No CPU fallback: every
// computation runs in the kernels of field.cu / ksg.cu / pearson.cu /
// pearson_gemm.cu; without a usable CUDA device calls return CORR_E_CUDA.
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <mutex>
#include <vector>

#include "sampler.cuh"

using namespace corr;

std::atomic<long long> corr::g_launch_count{0};

int corr::grid_waves_env() {
  static const int w = [] {
    const char* v = getenv("CORR_WAVES");
    return v ? atoi(v) : -1;  // -1: not set
  }();
  return w;
}

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, const char* detail = nullptr) {
  char buf[512];
  snprintf(buf, sizeof(buf), fmt, detail ? detail : "");
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
  g_last_error = buf;
  return CORR_E_CUDA;
}

// Makes `device` current for the scope of a call and restores the caller's device.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int device) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != device) err = cudaSetDevice(device);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void free_field(corr_field* f) {
  if (!f) return;
  for (int i = 0; i < 2; ++i) {
    if (f->stage[i]) cudaFree(f->stage[i]);
    if (f->ev_copied[i]) cudaEventDestroy(f->ev_copied[i]);
    if (f->ev_used[i]) cudaEventDestroy(f->ev_used[i]);
  }
  if (f->copy_st) cudaStreamDestroy(f->copy_st);
  cudaFree(f->F);
  cudaFree(f->Z);
  cudaFree(f->Zhi);
  cudaFree(f->Zlo);
  cudaFree(f->Zb);
  cudaFree(f->S);
  cudaFree(f->perm);
  cudaFree(f->cflag);
  cudaFree(f->spread);
  cudaFree(f->psi);
  cudaFree(f->err);
  cudaFree(f->tmaps);
  delete f;
}

// psi(m) = -gamma + sum_{t<m} 1/t at the integers m = 0..n+1 (psi(0) = NaN): the KSG
// arguments are integers, so the exact harmonic form replaces the paper's Lanczos
// approximation (reading R17).
std::vector<double> digamma_table(int n) {
  std::vector<double> t((size_t)n + 2);
  const double gamma = 0.57721566490153286060651209008240243;
  t[0] = NAN;
  double h = 0.0;
  for (int m = 1; m <= n + 1; ++m) {
    t[m] = h - gamma;
    h += 1.0 / (double)m;
  }
  return t;
}

// Allocates every device buffer of a field and uploads its psi table (stream-ordered).
int alloc_field(int32_t nx, int32_t ny, int32_t nz, int32_t members, int32_t device, cudaStream_t st,
                corr_field** out) {
  corr_field* f = new corr_field();
  memset(f, 0, sizeof(*f));
  f->device = device;
  f->nx = nx; f->ny = ny; f->nz = nz;
  f->n = members;
  f->n_pad = (members + 7) / 8 * 8;
  f->P = (int64_t)nx * ny * nz;
  const size_t row_elems = (size_t)f->P * f->n_pad;
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (cudaMalloc(p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  };
  if (!alloc((void**)&f->F, row_elems * 4) || !alloc((void**)&f->Z, row_elems * 4) ||
      !alloc((void**)&f->Zhi, row_elems * 4) || !alloc((void**)&f->Zlo, row_elems * 4) ||
      !alloc((void**)&f->Zb, row_elems * 2) ||
      !alloc((void**)&f->S, row_elems * 4) || !alloc((void**)&f->perm, row_elems * 2) ||
      !alloc((void**)&f->cflag, (size_t)f->P) || !alloc((void**)&f->spread, (size_t)f->P * 4) ||
      !alloc((void**)&f->psi, ((size_t)members + 2) * 8) || !alloc((void**)&f->err, 2 * sizeof(int))) {
    free_field(f);
    return fail(CORR_E_NOMEM, "device allocation failed for the field");
  }
  const std::vector<double> psi = digamma_table(members);
  cudaError_t e = cudaMemcpyAsync(f->psi, psi.data(), psi.size() * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(f->err, 0, 2 * sizeof(int), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // psi is a stack vector
  if (e != cudaSuccess) {
    free_field(f);
    return cuda_fail(e, "field allocation");
  }
  *out = f;
  return CORR_OK;
}

bool ksg_plus1(int32_t measure) { return (measure & CORR_F_KSG_PLUS1) != 0; }
KsgPath ksg_path(int32_t measure) {
  if (measure & CORR_F_KSG_DENSE) return kKsgDense;
  return (measure & CORR_F_KSG_SWEEP) ? kKsgSweep : kKsgAuto;
}

// Host-input staging of a field: two device slices of kStageMembers members each, a copy stream
// and the events ordering copies against transposes.  Created on the first host upload, kept for
// the field's lifetime (corr_field_update streams without allocating).
int ensure_staging(corr_field* f) {
  if (f->stage[0]) return CORR_OK;
  const size_t bytes = (size_t)kStageMembers * (size_t)f->P * 4;
  for (int i = 0; i < 2; ++i) {
    if (cudaMalloc((void**)&f->stage[i], bytes) != cudaSuccess) {
      cudaGetLastError();
      return fail(CORR_E_NOMEM, "device allocation failed for the host-upload staging slices");
    }
  }
  cudaError_t e = cudaStreamCreateWithFlags(&f->copy_st, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&f->ev_copied[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_used[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(e, "host-upload staging");
  return CORR_OK;
}

// Copies member-major values (host or device) into f and rebuilds every derived buffer on `st`.
// Host input is streamed: member slices of kStageMembers rows (contiguous in the [n][P] input,
// one cudaMemcpyAsync each) alternate between two device slices on the field's copy stream, and
// each slice is transposed into F on `st` as soon as it has landed, so the PCIe transfer overlaps
// the transposes (and, with pinned memory, whatever else runs on the device).  Non-finite values
// set err[1] bit 1 on the device; `sync` (corr_field_create) waits and reports them, otherwise
// (corr_field_update) the call returns at once and corr_check() reports them.
int ingest_values(corr_field* f, const float* values, cudaStream_t st, const char* who, bool sync) {
  cudaPointerAttributes attr;
  memset(&attr, 0, sizeof(attr));
  const cudaError_t pe = cudaPointerGetAttributes(&attr, values);
  if (pe != cudaSuccess) cudaGetLastError();
  const bool on_device = pe == cudaSuccess &&
                         (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) &&
                         attr.device == f->device;
  cudaError_t e = cudaMemsetAsync(f->err + 1, 0, sizeof(int), st);
  if (e == cudaSuccess && on_device) {
    e = launch_field_ingest(f, values, st);
  } else if (e == cudaSuccess) {
    const int rc = ensure_staging(f);
    if (rc) return rc;
    const size_t slice = (size_t)f->P * 4;  // bytes of one member row of the input
    for (int m0 = 0, i = 0; m0 < f->n && e == cudaSuccess; m0 += kStageMembers, ++i) {
      const int m1 = m0 + kStageMembers < f->n ? m0 + kStageMembers : f->n;
      const int b = i & 1;
      // the slice buffer is free once the transpose that last read it has run
      e = cudaStreamWaitEvent(f->copy_st, f->ev_used[b], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(f->stage[b], values + (size_t)m0 * f->P, (size_t)(m1 - m0) * slice,
                            cudaMemcpyHostToDevice, f->copy_st);
      if (e == cudaSuccess) e = cudaEventRecord(f->ev_copied[b], f->copy_st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, f->ev_copied[b], 0);
      if (e == cudaSuccess) e = launch_transpose_slice(f, f->stage[b], m0, m1, st);
      if (e == cudaSuccess) e = cudaEventRecord(f->ev_used[b], st);
    }
    if (e == cudaSuccess) e = launch_field_ingest(f, nullptr, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, who);
  if (!sync) return CORR_OK;
  int herr = 0;
  e = cudaMemcpyAsync(&herr, f->err + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, who);
  if (herr & 2) return fail(CORR_E_INVAL, "non-finite input value (SPEC.md:72)");
  return CORR_OK;
}

int check_pair_fields(const corr_field* fa, const corr_field*& fb) {
  if (!fa) return fail(CORR_E_INVAL, "field is NULL");
  if (!fb) fb = fa;
  if (fb->nx != fa->nx || fb->ny != fa->ny || fb->nz != fa->nz || fb->n != fa->n || fb->device != fa->device)
    return fail(CORR_E_INVAL, "fa and fb differ in dims, members or device");
  return CORR_OK;
}

int resolve_k(const corr_field* f, int32_t measure, int32_t& k) {
  const int kind = measure & 0xFF;
  if (kind != CORR_PEARSON && kind != CORR_KSG) return fail(CORR_E_INVAL, "unknown measure kind");
  if (measure & ~(0xFF | CORR_F_KSG_PLUS1 | CORR_F_ABS | CORR_F_KSG_DENSE | CORR_F_KSG_COUNT | CORR_F_KSG_SWEEP))
    return fail(CORR_E_INVAL, "unknown measure flags");
  if (kind == CORR_PEARSON) {
    k = 0;
    return CORR_OK;
  }
  const int n = f->n;
  if (n < 4) return fail(CORR_E_INVAL, "KSG needs at least 4 members (SPEC.md:184)");
  if (k == 0) {  // k = ceil(3n/100), clamped to [1, n-1]
    k = (3 * n + 99) / 100;
    if (k < 1) k = 1;
    if (k > n - 1) k = n - 1;
  }
  if (k < 1 || k > n - 1) return fail(CORR_E_INVAL, "k must be in [1, n-1]");
  return CORR_OK;
}

}  // namespace

extern "C" {

const char* corr_last_error(void) { return g_last_error.c_str(); }

int64_t corr_launch_count(void) { return (int64_t)g_launch_count.load(); }

int corr_ksg_comparisons(int32_t device, int64_t* count, int32_t reset) {
  if (!count) return fail(CORR_E_INVAL, "count is NULL");
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long v = 0;
  if (e == cudaSuccess) e = ksg_comparisons(&v, reset != 0);
  if (e != cudaSuccess) return cuda_fail(e, "corr_ksg_comparisons");
  *count = (int64_t)v;
  return CORR_OK;
}

int corr_ksg_nan_pairs(int32_t device, int64_t* count, int32_t reset) {
  if (!count) return fail(CORR_E_INVAL, "count is NULL");
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long v = 0;
  if (e == cudaSuccess) e = ksg_nan_pairs(&v, reset != 0);
  if (e != cudaSuccess) return cuda_fail(e, "corr_ksg_nan_pairs");
  *count = (int64_t)v;
  return CORR_OK;
}

}  // extern "C"

namespace corr {
namespace {
// Resident device copies of small host tables (region / tile lists), keyed by content (the lists
// are seed-free, so a context view's table is uploaded once).  No host synchronisation: the upload
// is stream-ordered on the first caller's stream and an event marks it ready; every user's stream
// waits on that event and records a last-use event.  Least-recently-used entries are evicted
// (freed stream-ordered after their last use) when the byte budget would be exceeded.
struct TableEntry {
  int device;
  uint64_t hash;
  std::vector<unsigned char> bytes;
  void* dptr;
  cudaEvent_t ready, last_use;
  uint64_t tick;
};
std::mutex g_table_mu;
std::vector<TableEntry> g_tables;
size_t g_table_bytes = 0;
uint64_t g_table_tick = 0;
constexpr size_t kTableCacheBytes = 64u << 20;
uint64_t fnv1a(const unsigned char* p, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}
}  // namespace

const void* cached_table(int device, const void* host, size_t bytes, cudaStream_t st) {
  const unsigned char* hp = static_cast<const unsigned char*>(host);
  const uint64_t h = fnv1a(hp, bytes);
  std::lock_guard<std::mutex> lock(g_table_mu);
  for (TableEntry& t : g_tables)
    if (t.device == device && t.hash == h && t.bytes.size() == bytes && memcmp(t.bytes.data(), hp, bytes) == 0) {
      if (cudaStreamWaitEvent(st, t.ready, 0) != cudaSuccess || cudaEventRecord(t.last_use, st) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      t.tick = ++g_table_tick;
      return t.dptr;
    }
  if (bytes > kTableCacheBytes) return nullptr;  // caller falls back to a per-call copy
  while (g_table_bytes + bytes > kTableCacheBytes) {  // evict this device's least recently used entry
    long lru = -1;
    for (size_t i = 0; i < g_tables.size(); ++i)
      if (g_tables[i].device == device && (lru < 0 || g_tables[i].tick < g_tables[(size_t)lru].tick)) lru = (long)i;
    if (lru < 0) return nullptr;  // the budget is held by other devices' tables: per-call copy
    TableEntry& t = g_tables[(size_t)lru];
    cudaStreamWaitEvent(st, t.last_use, 0);  // freed on this stream after its last use
    cudaFreeAsync(t.dptr, st);
    cudaEventDestroy(t.ready);
    cudaEventDestroy(t.last_use);
    g_table_bytes -= t.bytes.size();
    g_tables.erase(g_tables.begin() + lru);
  }
  TableEntry t{device, h, std::vector<unsigned char>(hp, hp + bytes), nullptr, nullptr, nullptr, ++g_table_tick};
  // stream-ordered upload; pageable host memory is consumed before cudaMemcpyAsync returns
  if (cudaMallocAsync(&t.dptr, bytes, st) != cudaSuccess ||
      cudaMemcpyAsync(t.dptr, host, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&t.last_use, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(t.ready, st) != cudaSuccess || cudaEventRecord(t.last_use, st) != cudaSuccess) {
    cudaGetLastError();
    if (t.dptr) cudaFreeAsync(t.dptr, st);
    if (t.ready) cudaEventDestroy(t.ready);
    if (t.last_use) cudaEventDestroy(t.last_use);
    return nullptr;
  }
  g_table_bytes += bytes;
  g_tables.push_back(std::move(t));
  return g_tables.back().dptr;
}
}  // namespace corr

extern "C" {

int corr_gemm_flops(int32_t device, int64_t* bf16_flops, int64_t* tf32_flops, int32_t reset) {
  if (!bf16_flops || !tf32_flops) return fail(CORR_E_INVAL, "output pointer is NULL");
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long v[2] = {0, 0};
  if (e == cudaSuccess) e = gemm_flops(v, reset != 0);
  if (e != cudaSuccess) return cuda_fail(e, "corr_gemm_flops");
  *bf16_flops = (int64_t)v[0];
  *tf32_flops = (int64_t)v[1];
  return CORR_OK;
}

int corr_field_create(const float* values, int32_t nx, int32_t ny, int32_t nz, int32_t members, int32_t device,
                      void* cuda_stream, corr_field** out) {
  if (!out) return fail(CORR_E_INVAL, "out is NULL");
  *out = nullptr;
  if (!values) return fail(CORR_E_INVAL, "values is NULL");
  if (nx < 1 || ny < 1 || nz < 1) return fail(CORR_E_INVAL, "grid dims must be >= 1");
  if (members < 2) return fail(CORR_E_INVAL, "members must be >= 2 (SPEC.md:34)");
  if (members > 4096) return fail(CORR_E_INVAL, "members > 4096 not supported (one pair is staged in shared memory)");
  int ndev = 0;
  const cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0) return cuda_fail(ce == cudaSuccess ? cudaErrorNoDevice : ce, "corr_field_create");
  if (device < 0 || device >= ndev) return fail(CORR_E_INVAL, "device ordinal out of range");
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  {
    // the per-call scratch (region tables, key arrays) comes from the stream-ordered pool: keep
    // freed blocks mapped instead of returning them to the OS at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = 64ull << 20;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }

  corr_field* f = nullptr;
  const int arc = alloc_field(nx, ny, nz, members, device, st, &f);
  if (arc) return arc;
  const int rc = ingest_values(f, values, st, "corr_field_create", true);
  if (rc) {
    free_field(f);
    return rc;
  }
  *out = f;
  return CORR_OK;
}

int corr_field_update(corr_field* f, const float* values, void* cuda_stream) {
  if (!f) return fail(CORR_E_INVAL, "field is NULL");
  if (!values) return fail(CORR_E_INVAL, "values is NULL");
  DeviceGuard guard(f->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  return ingest_values(f, values, (cudaStream_t)cuda_stream, "corr_field_update", false);
}

int corr_field_aggregate(const corr_field* f, int32_t fx, int32_t fy, int32_t fz, void* cuda_stream,
                         corr_field** out) {
  if (!out) return fail(CORR_E_INVAL, "out is NULL");
  *out = nullptr;
  if (!f) return fail(CORR_E_INVAL, "field is NULL");
  if (fx < 1 || fy < 1 || fz < 1) return fail(CORR_E_INVAL, "aggregation factors must be >= 1");
  DeviceGuard guard(f->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  corr_field* g = nullptr;
  const int rc = alloc_field((f->nx + fx - 1) / fx, (f->ny + fy - 1) / fy, (f->nz + fz - 1) / fz, f->n, f->device, st,
                             &g);
  if (rc) return rc;
  cudaError_t e = launch_field_aggregate(f, g, fx, fy, fz, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    free_field(g);
    return cuda_fail(e, "corr_field_aggregate");
  }
  *out = g;
  return CORR_OK;
}

int corr_field_destroy(corr_field* f) {
  if (!f) return CORR_OK;
  DeviceGuard guard(f->device);
  cudaDeviceSynchronize();
  free_field(f);
  return CORR_OK;
}

int corr_field_info(const corr_field* f, int32_t* nx, int32_t* ny, int32_t* nz, int32_t* members, int32_t* device) {
  if (!f) return fail(CORR_E_INVAL, "field is NULL");
  if (nx) *nx = f->nx;
  if (ny) *ny = f->ny;
  if (nz) *nz = f->nz;
  if (members) *members = f->n;
  if (device) *device = f->device;
  return CORR_OK;
}

static int eval_pairs_impl(const corr_field* fa, const corr_field* fb, int32_t measure, int32_t k,
                           const int64_t* idxA, const int64_t* idxB, int64_t npairs, float* out, float* dbg_eps,
                           int32_t* dbg_nx, int32_t* dbg_ny, void* cuda_stream) {
  int rc = check_pair_fields(fa, fb);
  if (rc) return rc;
  rc = resolve_k(fa, measure, k);
  if (rc) return rc;
  if (npairs < 0) return fail(CORR_E_INVAL, "npairs < 0");
  if (npairs == 0) return CORR_OK;
  if (!idxA || !idxB || !out) return fail(CORR_E_INVAL, "NULL index or output pointer");
  DeviceGuard guard(fa->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  PairSrc src;
  memset(&src, 0, sizeof(src));
  src.mode = kList;
  src.idxA = idxA;
  src.idxB = idxB;
  src.nunits = npairs;
  src.nx = fa->nx;
  src.ny = fa->ny;
  src.P = fa->P;
  src.same_field = fa == fb;
  src.err = fa->err;
  PairOut po;
  memset(&po, 0, sizeof(po));
  po.out = out;
  po.dbg_eps = dbg_eps;
  po.dbg_nx = dbg_nx;
  po.dbg_ny = dbg_ny;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cudaError_t e;
  if ((measure & 0xFF) == CORR_KSG) {
    e = launch_ksg(fa, fb, k, ksg_plus1(measure), ksg_path(measure), (measure & CORR_F_KSG_COUNT) != 0, src, po, st);
    if (e == cudaErrorNotSupported) return fail(CORR_E_INVAL, "KSG configuration not supported");
  } else {
    e = launch_pearson_pairs(fa, fb, src, po, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "corr_eval_pairs");
  return CORR_OK;
}

int corr_eval_pairs(const corr_field* fa, const corr_field* fb, int32_t measure, int32_t k, const int64_t* idxA,
                    const int64_t* idxB, int64_t npairs, float* out, void* cuda_stream) {
  return eval_pairs_impl(fa, fb, measure, k, idxA, idxB, npairs, out, nullptr, nullptr, nullptr, cuda_stream);
}

int corr_ksg_debug(const corr_field* fa, const corr_field* fb, int32_t k, const int64_t* idxA, const int64_t* idxB,
                   int64_t npairs, float* eps, int32_t* nx, int32_t* ny, void* cuda_stream) {
  if (!eps || !nx || !ny) return fail(CORR_E_INVAL, "NULL debug output pointer");
  if (!fa) return fail(CORR_E_INVAL, "field is NULL");
  if (npairs <= 0) return npairs == 0 ? CORR_OK : fail(CORR_E_INVAL, "npairs < 0");
  DeviceGuard guard(fa->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  float* tmp = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&tmp, (size_t)npairs * 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "corr_ksg_debug");
  const int rc = eval_pairs_impl(fa, fb, CORR_KSG, k, idxA, idxB, npairs, tmp, eps, nx, ny, cuda_stream);
  cudaFreeAsync(tmp, st);
  return rc;
}

int corr_region_max(const corr_field* fa, const corr_field* fb, int32_t measure, int32_t k, const corr_box* regionA,
                    const corr_box* regionB, int64_t nregion_pairs, int64_t samples, uint64_t seed, float* out_max,
                    int64_t* out_argmax, void* cuda_stream) {
  const corr_field* fb_in = fb;
  int rc = check_pair_fields(fa, fb);
  if (rc) return rc;
  rc = resolve_k(fa, measure, k);
  if (rc) return rc;
  if (nregion_pairs < 0) return fail(CORR_E_INVAL, "nregion_pairs < 0");
  if (nregion_pairs == 0) return CORR_OK;
  if (!regionA || !regionB || !out_max || !out_argmax) return fail(CORR_E_INVAL, "NULL region or output pointer");
  if (samples < 0 || samples >= (int64_t)1 << 32) return fail(CORR_E_INVAL, "samples must be in [0, 2^32)");
  std::vector<RegionDev> reg((size_t)nregion_pairs);
  int64_t total = 0;
  for (int64_t r = 0; r < nregion_pairs; ++r) {
    const corr_box* bx[2] = {&regionA[r], &regionB[r]};
    for (int s = 0; s < 2; ++s) {
      const corr_box& b = *bx[s];
      if (b.x1 <= b.x0 || b.y1 <= b.y0 || b.z1 <= b.z0) return fail(CORR_E_INVAL, "empty region box");
      if (b.x0 < 0 || b.y0 < 0 || b.z0 < 0 || b.x1 > fa->nx || b.y1 > fa->ny || b.z1 > fa->nz)
        return fail(CORR_E_RANGE, "region box outside the grid");
    }
    RegionDev& R = reg[(size_t)r];
    R.A = regionA[r];
    R.B = regionB[r];
    R.nA = (int64_t)(R.A.x1 - R.A.x0) * (R.A.y1 - R.A.y0) * (R.A.z1 - R.A.z0);
    R.nB = (int64_t)(R.B.x1 - R.B.x0) * (R.B.y1 - R.B.y0) * (R.B.z1 - R.B.z0);
    R.off = total;
    if (samples == 0 && R.nA * R.nB >= ((int64_t)1 << 32))
      return fail(CORR_E_INVAL, "exhaustive region pair with |A|*|B| >= 2^32");
    total += samples > 0 ? samples : R.nA * R.nB;
  }
  DeviceGuard guard(fa->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  RegionDev* dreg = nullptr;
  unsigned long long* keys = nullptr;
  // the region table: resident device copy reused across calls with the same regions (context view)
  const size_t reg_bytes = reg.size() * sizeof(RegionDev);
  dreg = const_cast<RegionDev*>(static_cast<const RegionDev*>(cached_table(fa->device, reg.data(), reg_bytes, st)));
  const bool own_reg = dreg == nullptr;
  cudaError_t e = cudaSuccess;
  if (own_reg) e = cudaMallocAsync((void**)&dreg, reg_bytes, st);
  uint64_t* rkey = nullptr;  // sampler keys of this call's seed, derived on the device
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&keys, (size_t)nregion_pairs * 8, st);
  if (e == cudaSuccess && samples > 0) e = cudaMallocAsync((void**)&rkey, (size_t)nregion_pairs * 8, st);
  if (e != cudaSuccess) return cuda_fail(e, "corr_region_max alloc");
  if (own_reg) e = cudaMemcpyAsync(dreg, reg.data(), reg_bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(keys, 0, (size_t)nregion_pairs * 8, st);
  if (e == cudaSuccess && rkey) e = launch_region_keys(dreg, nregion_pairs, seed, rkey, st);

  PairSrc src;
  memset(&src, 0, sizeof(src));
  src.mode = samples > 0 ? kSampled : kExhaustive;
  src.reg = dreg;
  src.rkey = rkey;
  src.nreg = nregion_pairs;
  src.samples = samples;
  src.nunits = total;
  src.nx = fa->nx;
  src.ny = fa->ny;
  src.P = fa->P;
  src.same_field = (fb_in == nullptr || fb_in == fa);
  src.err = fa->err;
  PairOut po;
  memset(&po, 0, sizeof(po));
  po.keys = keys;
  po.absval = (measure & CORR_F_ABS) != 0;
  if (e == cudaSuccess) {
    if ((measure & 0xFF) == CORR_KSG) {
      e = launch_ksg(fa, fb, k, ksg_plus1(measure), ksg_path(measure), (measure & CORR_F_KSG_COUNT) != 0, src, po, st);
      if (e == cudaErrorNotSupported) {
        if (own_reg) cudaFreeAsync(dreg, st);
        cudaFreeAsync(keys, st);
        if (rkey) cudaFreeAsync(rkey, st);
        return fail(CORR_E_INVAL, "KSG configuration not supported");
      }
    } else if (samples == 0) {
      e = launch_pearson_block(fa, fb, reg.data(), dreg, nregion_pairs, po.absval, keys, st);
      if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        e = launch_pearson_pairs(fa, fb, src, po, st);
      }
    } else {
      e = launch_pearson_pairs(fa, fb, src, po, st);
    }
  }
  if (e == cudaSuccess) e = launch_region_finalize(src, keys, out_max, out_argmax, st);
  if (own_reg) cudaFreeAsync(dreg, st);
  cudaFreeAsync(keys, st);
  if (rkey) cudaFreeAsync(rkey, st);
  if (e != cudaSuccess) return cuda_fail(e, "corr_region_max");
  return CORR_OK;
}

int corr_check(const corr_field* f, void* cuda_stream) {
  if (!f) return fail(CORR_E_INVAL, "field is NULL");
  DeviceGuard guard(f->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "corr_check");
  int h[2] = {0, 0};
  e = cudaMemcpy(h, f->err, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "corr_check");
  if (h[1] & 2) {
    const int zero = 0;
    cudaMemcpy(f->err + 1, &zero, sizeof(int), cudaMemcpyHostToDevice);
    return fail(CORR_E_INVAL, "non-finite input value in an earlier corr_field_update (SPEC.md:72)");
  }
  if (h[0] & 1) {
    const int zero = 0;
    cudaMemcpy(f->err, &zero, sizeof(int), cudaMemcpyHostToDevice);
    return fail(CORR_E_RANGE, "point index out of range in an earlier call");
  }
  return CORR_OK;
}

}  // extern "C"
