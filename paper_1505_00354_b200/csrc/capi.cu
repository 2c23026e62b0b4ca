// The C ABI (include/fastleg_b200.h): argument validation in the reference's
// order with its messages, host/device staging, per-call stream-ordered
// scratch, and the TransformConfig-equivalent device plan.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "czt.cuh"
#include "direct.cuh"
#include "fast_ndct.cuh"
#include "launch.cuh"
#include "dense_gemv.cuh"
#include "dist_ndct.cuh"
#include "l2c_asy.cuh"
#include "l2c_fast.cuh"
#include "l2c_ozaki.cuh"
#include "leg2cheb.cuh"

namespace flb {

namespace {
thread_local std::string g_last_error;
std::atomic<int> g_free_mode{FL_NDCT_FAST};  // fl_set_free_ndct_mode
std::atomic<unsigned long long> g_launches{0};
}  // namespace

void fail(fl_status s, const std::string& msg) { throw Error{s, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{FL_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")"};
  }
}

void note_launch(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cuda_check(cudaGetLastError(), name);
}

namespace {

template <class F>
fl_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return FL_OK;
  } catch (const Error& e) {
    g_last_error = e.message;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "fastleg_b200: host allocation failed";
    return FL_RUNTIME_ERROR;
  } catch (...) {
    g_last_error = "fastleg_b200: unknown error";
    return FL_RUNTIME_ERROR;
  }
}

void require_device() {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(FL_CUDA_ERROR, std::string("fastleg_b200: no usable CUDA device (") +
                            (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") +
                            "); there is no CPU fallback");
  }
  // Keep stream-ordered scratch cached across calls: the default pool would
  // otherwise unmap it at every synchronize (re-mapping GiBs per call).
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && !done[dev]) {
    cudaMemPool_t pool;
    FLB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t threshold = UINT64_MAX;
    FLB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    done[dev] = true;
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  const cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// page-locked (cudaHostAlloc / cudaHostRegister) host memory: the only host
// memory an async copy can overlap with kernels
bool is_pinned_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  const cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// A column block (n rows x batch columns, stride ld) as a device pointer.
struct DevIn {
  const double* ptr = nullptr;
  size_t ld = 0;
  double* owned = nullptr;
  cudaStream_t s;
  DevIn(const double* user, size_t n, size_t batch, size_t ld_user, cudaStream_t st) : s(st) {
    if (is_device_ptr(user)) {
      ptr = user;
      ld = ld_user;
      return;
    }
    const size_t bytes = n * batch * sizeof(double);
    FLB_CUDA(cudaMallocAsync(&owned, bytes ? bytes : 8, s));
    if (bytes)
      FLB_CUDA(cudaMemcpy2DAsync(owned, n * sizeof(double), user, ld_user * sizeof(double),
                                 n * sizeof(double), batch, cudaMemcpyHostToDevice, s));
    ptr = owned;
    ld = n;
  }
  ~DevIn() {
    if (owned) cudaFreeAsync(owned, s);
  }
};

struct DevOut {
  double* ptr = nullptr;
  size_t ld = 0;
  double* user;
  size_t n, batch, ld_user;
  bool host;
  cudaStream_t s;
  DevOut(double* u, size_t n_, size_t batch_, size_t ld_u, cudaStream_t st)
      : user(u), n(n_), batch(batch_), ld_user(ld_u), s(st) {
    host = u != nullptr && !is_device_ptr(u);
    if (!host) {  // device pointer, or an output the caller does not want (null)
      ptr = u;
      ld = ld_u;
      return;
    }
    const size_t bytes = n * batch * sizeof(double);
    FLB_CUDA(cudaMallocAsync(&ptr, bytes ? bytes : 8, s));
    ld = n;
  }
  void finish() {
    if (host && n * batch)
      FLB_CUDA(cudaMemcpy2DAsync(user, ld_user * sizeof(double), ptr, n * sizeof(double),
                                 n * sizeof(double), batch, cudaMemcpyDeviceToHost, s));
  }
  ~DevOut() {
    if (host && ptr) cudaFreeAsync(ptr, s);
  }
};

template <class T>
struct DevScratch {
  T* p = nullptr;
  cudaStream_t s;
  DevScratch(size_t count, cudaStream_t st) : s(st) {
    FLB_CUDA(cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), s));
  }
  ~DevScratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

void sync(cudaStream_t s) { FLB_CUDA(cudaStreamSynchronize(s)); }

// The non-finite flag of one synchronous call: a pinned, mapped host int of
// the calling host thread (a few per thread, for nested calls), zeroed by the
// host before the call's kernels are enqueued, raised by the kernels through
// its device alias, and read after the call's stream synchronisation -- no
// allocation, memset or device-to-host copy per call (they were about a third
// of a single-column N = 1024 DLT's 33 us).
struct SyncFlag {
  int* p = nullptr;  // what the kernels write (device alias of the host int)
  SyncFlag() {
    Slots& t = slots();
    if (t.depth >= kDepth) fail(FL_RUNTIME_ERROR, "fastleg: flag nesting too deep");
    if (!t.h) {
      void* mem = nullptr;
      FLB_CUDA(cudaHostAlloc(&mem, kDepth * sizeof(int), cudaHostAllocPortable | cudaHostAllocMapped));
      t.h = static_cast<volatile int*>(mem);
    }
    h_ = t.h + t.depth++;
    *h_ = 0;
    void* dp = nullptr;
    FLB_CUDA(cudaHostGetDevicePointer(&dp, const_cast<int*>(h_), 0));
    p = static_cast<int*>(dp);
  }
  ~SyncFlag() { --slots().depth; }
  SyncFlag(const SyncFlag&) = delete;
  SyncFlag& operator=(const SyncFlag&) = delete;
  // synchronises the stream; true if a kernel raised the flag
  bool wait(cudaStream_t s) {
    sync(s);
    return *h_ != 0;
  }

 private:
  static constexpr int kDepth = 8;
  struct Slots {
    volatile int* h = nullptr;
    int depth = 0;
    ~Slots() {
      if (h) cudaFreeHost(const_cast<int*>(h));
    }
  };
  static Slots& slots() {
    thread_local Slots t;
    return t;
  }
  volatile int* h_ = nullptr;
};

const char* trig_name(int op) {
  switch (op) {
    case FL_DCT_III: return "dct_iii";
    case FL_DST_III: return "dst_iii";
    case FL_DCT_III_T: return "dct_iii_transpose";
    default: return "dst_iii_transpose";
  }
}

void check_kind(int kind) {
  if (kind != FL_CHEB1 && kind != FL_CHEBSTAR) fail(FL_INVALID_ARGUMENT, "fastleg: unknown grid kind");
}

void check_ld(size_t n, size_t ld, size_t batch) {
  if (batch > 1 && ld < n) fail(FL_INVALID_ARGUMENT, "fastleg: column stride smaller than size");
}

// ndct.hpp:49-59 min_taylor_terms
int min_taylor_terms(int kind, double tolerance) {
  if (!(tolerance > 0.0 && tolerance < 1.0))
    fail(FL_INVALID_ARGUMENT, "min_taylor_terms: tolerance must lie in (0, 1)");
  const double q = kind == FL_CHEB1 ? 0.83845 : 1.0 / (6.0 * kPi);
  double bound = 1.0;
  for (int l = 1; l <= 30; ++l) {
    bound *= q / static_cast<double>(l);
    if (bound <= tolerance) return l;
  }
  fail(FL_DOMAIN_ERROR, "min_taylor_terms: tolerance unattainable with <= 30 terms");
}

bool overflow_guard(size_t n, int num_terms) {  // ndct.hpp:87-88
  return n > 1 && static_cast<double>(num_terms - 1) * std::log10(static_cast<double>(n - 1)) > 300.0;
}

__global__ void nonfinite_kernel(const double* __restrict__ v, size_t n, size_t batch, size_t ld,
                                 const double* __restrict__ mult, int* flag) {
  const size_t total = n * batch;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t col = i / n, row = i % n;
    double x = v[col * ld + row];
    if (mult) x *= mult[row];
    if (!isfinite(x)) atomicOr(flag, 1);
  }
}

// one CTA: r[0] = max_k |delta_k|, r[1] = sum_k |c_k| (fixed reduction order)
__global__ void maxabs_l1_kernel(const double* __restrict__ d, size_t nd,
                                 const double* __restrict__ c, size_t nc, double* r) {
  __shared__ double sm[2][1024];
  double m = 0.0, s = 0.0;
  for (size_t i = threadIdx.x; i < nd; i += blockDim.x) m = fmax(m, fabs(d[i]));
  for (size_t i = threadIdx.x; i < nc; i += blockDim.x) s += fabs(c[i]);
  sm[0][threadIdx.x] = m;
  sm[1][threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sm[0][threadIdx.x] = fmax(sm[0][threadIdx.x], sm[0][threadIdx.x + w]);
      sm[1][threadIdx.x] += sm[1][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    r[0] = sm[0][0];
    r[1] = sm[1][0];
  }
}

void reduce_maxabs_l1(const double* d, size_t nd, const double* c, size_t nc, double* r,
                      cudaStream_t s) {
  maxabs_l1_kernel<<<1, 1024, 0, s>>>(d, nd, c, nc, r);
  note_launch("maxabs_l1_kernel");
}

bool any_nonfinite(const double* v, size_t n, size_t batch, size_t ld, const double* mult,
                   cudaStream_t s) {
  SyncFlag flag;
  nonfinite_kernel<<<sm_count() * 4, 256, 0, s>>>(v, n, batch, ld, mult, flag.p);
  note_launch("nonfinite_kernel");
  const bool h = flag.wait(s);
  return h != 0;
}

// Enqueues an NDCT (literal kind, or the fast cheb1 path); non-finite inputs
// raise *flag (device int, zeroed by the caller). Callers check
// overflow_guard first.
void enqueue_ndct(int transpose, int kind, size_t n, int num_terms, const double* delta,
                  const double* in, size_t ld_in, double* out, size_t ld_out, size_t batch,
                  const double* in_mult, const FastNdct* fast, int* flag, cudaStream_t s) {
  if (num_terms <= 0) {
    FLB_CUDA(cudaMemset2DAsync(out, ld_out * sizeof(double), 0, n * sizeof(double), batch, s));
    nonfinite_kernel<<<sm_count() * 4, 256, 0, s>>>(in, n, batch, ld_in, in_mult, flag);
    note_launch("nonfinite_kernel");
  } else if (fast) {
    fast_ndct_run(*fast, transpose, in, ld_in, out, ld_out, batch, in_mult, flag, s);
  } else {
    if (ld_in != ld_out && batch > 1)
      fail(FL_RUNTIME_ERROR, "ndct: mismatched strides");  // internal: callers pass equal ld
    czt_ndct(transpose, kind, n, num_terms, delta, in, out, batch, ld_in, in_mult, flag, s);
  }
}

// Runs an NDCT with the reference's validation order: non-finite
// (invalid_argument) before overflow.
void run_ndct(const char* where, int transpose, int kind, size_t n, int num_terms,
              const double* delta, const double* in, size_t ld_in, double* out, size_t ld_out,
              size_t batch, const double* in_mult, const FastNdct* fast, cudaStream_t s) {
  if (overflow_guard(n, num_terms)) {
    if (any_nonfinite(in, n, batch, ld_in, in_mult, s))
      fail(FL_INVALID_ARGUMENT, std::string(where) + ": non-finite input");
    fail(FL_OVERFLOW_ERROR, std::string(where) + ": n^l exceeds double range");
  }
  SyncFlag flag;
  enqueue_ndct(transpose, kind, n, num_terms, delta, in, ld_in, out, ld_out, batch, in_mult, fast,
               flag.p, s);
  const bool h = flag.wait(s);
  if (h) fail(FL_INVALID_ARGUMENT, std::string(where) + ": non-finite input");
}

// The NDCT inside dlt/idlt without a host round trip of its own: the
// non-finite flag is read once, after everything else, by finish (whose stream
// synchronisation is the call's only one).
struct DeferredNdct {
  SyncFlag flag;
  explicit DeferredNdct(cudaStream_t) {}
  void run(const char* where, int transpose, int kind, size_t n, int num_terms,
           const double* delta, const double* in, size_t ld_in, double* out, size_t ld_out,
           size_t batch, const double* in_mult, const FastNdct* fast, cudaStream_t s) {
    if (overflow_guard(n, num_terms)) {  // the reference's order: non-finite, then overflow
      run_ndct(where, transpose, kind, n, num_terms, delta, in, ld_in, out, ld_out, batch,
               in_mult, fast, s);
      return;
    }
    enqueue_ndct(transpose, kind, n, num_terms, delta, in, ld_in, out, ld_out, batch, in_mult,
                 fast, flag.p, s);
    where_ = where;
  }
  void finish(cudaStream_t s) {
    const bool h = flag.wait(s);
    if (h) fail(FL_INVALID_ARGUMENT, std::string(where_) + ": non-finite input");
  }
  const char* where_ = "ndct_apply";
};

// ---- host-buffer pipeline ------------------------------------------------
// A transform of host columns (host in, host out) is cut into column chunks
// that flow through three streams -- H2D copy | compute | D2H copy -- with three
// device buffer sets, so both PCIe directions and the kernels overlap. The
// non-finite flags of all chunks are checked once at the end.
struct PipeStreams {
  cudaStream_t h2d, comp, d2h;
};

const PipeStreams& pipe_streams(int dev) {
  static std::mutex mu;
  static std::map<int, PipeStreams> per_dev;
  std::lock_guard<std::mutex> lock(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    PipeStreams ps;
    FLB_CUDA(cudaStreamCreateWithFlags(&ps.h2d, cudaStreamNonBlocking));
    FLB_CUDA(cudaStreamCreateWithFlags(&ps.comp, cudaStreamNonBlocking));
    FLB_CUDA(cudaStreamCreateWithFlags(&ps.d2h, cudaStreamNonBlocking));
    it = per_dev.emplace(dev, ps).first;
  }
  return it->second;
}

#ifndef FLB_PIPE_CHUNKS
#define FLB_PIPE_CHUNKS 32
#endif
constexpr size_t kPipeMinBytes = size_t(64) << 20;  // below this one copy each way is as fast

// Only pinned host buffers: a D2H copy into pageable memory blocks the host
// until the chunk's compute is done, which would serialise the pipeline
// (pageable buffers take the one-copy-each-way path instead).
bool pipeline_ok(const double* in, const double* out, size_t n, size_t batch) {
  return is_pinned_host(in) && is_pinned_host(out) && batch >= 8 &&
         n * batch * sizeof(double) >= kPipeMinBytes;
}

// compute(din, dout, cols, flag, stream): device columns of stride n.
template <class F>
void run_pipelined(int dev, size_t n, const double* in, double* out, size_t batch, size_t ld,
                   cudaStream_t user, const char* where, F&& compute) {
  constexpr int NB = 3;  // buffer sets: H2D of chunk i + 3 waits for the D2H of chunk i
  const PipeStreams& ps = pipe_streams(dev);
  const size_t chunks = std::max<size_t>(1, std::min<size_t>(FLB_PIPE_CHUNKS, batch / 256));
  const size_t per = (batch + chunks - 1) / chunks;
  DevScratch<double> din(NB * per * n, user), dout(NB * per * n, user);
  DevScratch<int> flags(chunks, user);
  FLB_CUDA(cudaMemsetAsync(flags.p, 0, chunks * sizeof(int), user));
  cudaEvent_t start, h2d[NB], comp[NB], d2h[NB];
  FLB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  for (int b = 0; b < NB; ++b)
    for (cudaEvent_t* e : {&h2d[b], &comp[b], &d2h[b]})
      FLB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  FLB_CUDA(cudaEventRecord(start, user));  // buffers allocated / flags zeroed on `user`
  for (cudaStream_t st : {ps.h2d, ps.comp, ps.d2h}) FLB_CUDA(cudaStreamWaitEvent(st, start, 0));
  for (size_t i = 0; i < chunks; ++i) {
    const size_t c0 = i * per;
    if (c0 >= batch) break;
    const size_t cols = std::min(per, batch - c0);
    const int b = (int)(i % NB);
    double* di = din.p + b * per * n;
    double* dq = dout.p + b * per * n;
    if (i >= (size_t)NB) FLB_CUDA(cudaStreamWaitEvent(ps.h2d, d2h[b], 0));
    FLB_CUDA(cudaMemcpy2DAsync(di, n * 8, in + c0 * ld, ld * 8, n * 8, cols,
                               cudaMemcpyHostToDevice, ps.h2d));
    FLB_CUDA(cudaEventRecord(h2d[b], ps.h2d));
    FLB_CUDA(cudaStreamWaitEvent(ps.comp, h2d[b], 0));
    compute(di, dq, cols, flags.p + i, ps.comp);
    FLB_CUDA(cudaEventRecord(comp[b], ps.comp));
    FLB_CUDA(cudaStreamWaitEvent(ps.d2h, comp[b], 0));
    FLB_CUDA(cudaMemcpy2DAsync(out + c0 * ld, ld * 8, dq, n * 8, n * 8, cols,
                               cudaMemcpyDeviceToHost, ps.d2h));
    FLB_CUDA(cudaEventRecord(d2h[b], ps.d2h));
  }
  std::vector<int> h(chunks, 0);
  FLB_CUDA(cudaStreamSynchronize(ps.comp));
  FLB_CUDA(cudaStreamSynchronize(ps.d2h));
  FLB_CUDA(cudaStreamSynchronize(ps.h2d));
  // the scratch frees below are ordered on `user`: make it follow the pipeline
  FLB_CUDA(cudaMemcpyAsync(h.data(), flags.p, chunks * sizeof(int), cudaMemcpyDeviceToHost, user));
  sync(user);
  cudaEventDestroy(start);
  for (int b = 0; b < NB; ++b)
    for (cudaEvent_t e : {h2d[b], comp[b], d2h[b]}) cudaEventDestroy(e);
  for (int v : h)
    if (v) fail(FL_INVALID_ARGUMENT, std::string(where) + ": non-finite input");
}

}  // namespace
}  // namespace flb

using namespace flb;

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct fl_plan {
  size_t n = 0;
  double tolerance = 0.0;
  int kind = FL_CHEBSTAR;
  int num_terms = 0;
  int mode = FL_NDCT_FAST;
  int device = 0;
  double* theta = nullptr;   // n
  double* x = nullptr;       // n
  double* w = nullptr;       // n
  double* tstar = nullptr;   // n (plan kind)
  double* delta = nullptr;   // n (plan kind)
  double* lambda = nullptr;  // n  (LambdaCache(n - 1))
  double* s = nullptr;       // n  (scaled Lambda)
  FastNdct* fast = nullptr;  // cheb1-internal NDCT (power-of-two n), or null
  L2CFast* l2c = nullptr;    // Toeplitz-Hankel leg2cheb (n >= kL2CFastMin), or null
  int l2c_mode = 1;          // 1: fast conversion for few columns when available; 0: direct;
                             // 2: asymptotic expansion (power-of-two n), else as 1
  L2CAsy* asy = nullptr;     // asymptotic-expansion leg2cheb (lazy, mode 2)
  int gemm_mode = FL_GEMM_INT8_SPLIT;  // arithmetic of the direct conversion product
  L2COzaki* oz[2] = {nullptr, nullptr};  // split-int8 slices of M, (m + 1/2) M^T (lazy)
  int dlt_method = FL_DLT_DIRECT;        // dlt/idlt: dense product where supported
  L2COzaki* dense[2] = {nullptr, nullptr};  // split-int8 slices of P, (m + 1/2) P^T (lazy)
  DenseGemv* gemv = nullptr;                // fp64 table of P for <= 16 columns (lazy)
  std::mutex mu;
};

namespace {

void plan_free(fl_plan* p) {
  for (double* q : {p->theta, p->x, p->w, p->tstar, p->delta, p->lambda, p->s})
    if (q) cudaFree(q);
  if (p->fast) fast_ndct_destroy(p->fast);
  if (p->l2c) l2c_fast_destroy(p->l2c);
  if (p->asy) l2c_asy_destroy(p->asy);
  for (L2COzaki* o : p->oz) l2c_ozaki_destroy(o);
  for (L2COzaki* o : p->dense) l2c_ozaki_destroy(o);
  if (p->gemv) dense_gemv_destroy(p->gemv);
  delete p;
}

void plan_finish(fl_plan* p) {
  const size_t n = p->n;
  FLB_CUDA(cudaMalloc(&p->tstar, n * 8));
  FLB_CUDA(cudaMalloc(&p->delta, n * 8));
  FLB_CUDA(cudaMalloc(&p->lambda, n * 8));
  FLB_CUDA(cudaMalloc(&p->s, n * 8));
  launch_reference_grid(n, p->kind, p->theta, p->tstar, p->delta, 0);
  launch_lambda(n - 1, p->lambda, 0);
  scaled_lambda(p->lambda, p->s, n, 0);
  p->fast = fast_ndct_create(n, p->tolerance, p->kind, p->delta);
  FLB_CUDA(cudaDeviceSynchronize());
}

// The split-int8 conversion product for this call, or null (fp64 path).
const L2COzaki* plan_ozaki(fl_plan* p, int transpose, size_t batch, cudaStream_t s) {
  if (p->gemm_mode != FL_GEMM_INT8_SPLIT || batch <= 16 || !l2c_ozaki_supported(p->n) ||
      p->n > 16384)
    return nullptr;
  std::lock_guard<std::mutex> lock(p->mu);
  if (!p->oz[transpose]) {
    // the A digits are written on `s`: publish the product only once they are
    // complete, so a caller on another stream never reads them half-written
    // (TransformConfig is shared across threads, transforms.hpp:15-18)
    L2COzaki* oz = l2c_ozaki_create(p->n, p->s, transpose, transpose, s);
    FLB_CUDA(cudaStreamSynchronize(s));
    p->oz[transpose] = oz;
  }
  return p->oz[transpose];
}

// The direct product for this call (fl_dlt: P, fl_idlt: (m + 1/2) P^T), or
// null (factored path): > 16 columns, the int8-split arithmetic, n a
// multiple of 256 in [512, 8192]. Built once per plan and direction, on
// first use, published after its digits are complete (as plan_ozaki).
const L2COzaki* plan_dense(fl_plan* p, int idlt, size_t batch, cudaStream_t s) {
  if (p->dlt_method != FL_DLT_DIRECT || p->gemm_mode != FL_GEMM_INT8_SPLIT || batch <= 16 ||
      !l2c_dense_supported(p->n))
    return nullptr;
  std::lock_guard<std::mutex> lock(p->mu);
  if (!p->dense[idlt]) {
    L2COzaki* d = l2c_dense_create(p->n, p->kind, p->delta, idlt, s);
    FLB_CUDA(cudaStreamSynchronize(s));
    p->dense[idlt] = d;
  }
  return p->dense[idlt];
}

// The plan's Toeplitz-Hankel factors (n >= 2^14), built on first use: plans
// whose conversion is the asymptotic expansion (power-of-two n >= 2^20) never
// pay the pivoted Cholesky (0.24 s at 2^26).
L2CFast* plan_th(const fl_plan* cp, cudaStream_t s) {
  fl_plan* p = const_cast<fl_plan*>(cp);
  if (p->n < kL2CFastMin) return nullptr;
  std::lock_guard<std::mutex> lock(p->mu);
  if (!p->l2c) {
    L2CFast* f = l2c_fast_create(p->n, p->s, s);
    FLB_CUDA(cudaStreamSynchronize(s));
    p->l2c = f;
  }
  return p->l2c;
}

// The direct method for <= 16 columns (fl_dlt / fl_idlt): fp64 products over
// the plan's table of P_n(x_k), N even in [256, 8192] (built on first use,
// published once complete, as plan_dense).
const DenseGemv* plan_gemv(fl_plan* p, size_t batch, cudaStream_t s) {
  if (p->dlt_method != FL_DLT_DIRECT || batch > 16 || !dense_gemv_supported(p->n)) return nullptr;
  std::lock_guard<std::mutex> lock(p->mu);
  if (!p->gemv) {
    DenseGemv* g = dense_gemv_create(p->n, p->kind, p->delta, s);
    FLB_CUDA(cudaStreamSynchronize(s));
    p->gemv = g;
  }
  return p->gemv;
}

// The asymptotic-expansion conversion of the plan (built on first use and
// published once its tables are complete, as plan_ozaki).
const L2CAsy* plan_asy(fl_plan* p, cudaStream_t s) {
  if (!l2c_asy_supported(p->n)) return nullptr;
  std::lock_guard<std::mutex> lock(p->mu);
  if (!p->asy) {
    L2CAsy* a = l2c_asy_create(p->n, p->s, s);
    FLB_CUDA(cudaStreamSynchronize(s));
    p->asy = a;
  }
  return p->asy;
}

// Whether the plan converts `batch` columns by the asymptotic expansion.
bool plan_wants_asy(const fl_plan* p, size_t batch) {
  return l2c_asy_supported(p->n) && batch <= kL2CFastMaxCols &&
         (p->l2c_mode == FL_LEG2CHEB_ASYMPTOTIC ||
          (p->l2c_mode == FL_LEG2CHEB_FAST && p->n >= kL2CAsyMin));
}

// The plan's conversion product (transforms.hpp:47 / :62): chat = M in, or
// (m + 1/2) M^T in for the inverse; device columns of stride n.
// in: columns of stride n; out: stride ld_out. The conversion kernels take a
// single column stride for both, so a strided output goes through a
// stride-n scratch.
void plan_convert(fl_plan* p, int transpose, const double* in, double* out, size_t batch,
                  size_t ld_out, cudaStream_t s) {
  const size_t n = p->n;
  if (ld_out != n) {
    DevScratch<double> t(n * batch, s);
    plan_convert(p, transpose, in, t.p, batch, n, s);
    FLB_CUDA(cudaMemcpy2DAsync(out, ld_out * 8, t.p, n * 8, n * 8, batch,
                               cudaMemcpyDeviceToDevice, s));
    return;
  }
  // FAST: the asymptotic expansion where it beats Toeplitz-Hankel (power-of-two
  // n >= 2^16: 0.15 vs 0.19 ms there, 1.75 vs 2.86 ms at 2^20, 142 vs 288 ms
  // at 2^26), else Toeplitz-Hankel
  const L2CAsy* asy = plan_wants_asy(p, batch) ? plan_asy(p, s) : nullptr;
  if (asy)
    l2c_asy_apply(*asy, transpose, in, out, batch, n, transpose, s);
  else if (p->l2c_mode != FL_LEG2CHEB_DIRECT && batch <= kL2CFastMaxCols && plan_th(p, s))
    l2c_fast_apply(*plan_th(p, s), transpose, in, out, batch, n, transpose, s);
  else if (const L2COzaki* oz = plan_ozaki(p, transpose, batch, s))
    l2c_ozaki_apply(*oz, in, out, batch, n, s);
  else
    leg2cheb_direct(transpose, n, p->s, in, out, batch, n, transpose, s);
}

}  // namespace

extern "C" {

const char* fl_last_error(void) { return g_last_error.c_str(); }

int fl_device_available(void) {
  return guarded([] { require_device(); }) == FL_OK ? 1 : 0;
}

uint64_t fl_kernel_launch_count(void) { return g_launches.load(); }

fl_status fl_set_free_ndct_mode(int mode) {
  return guarded([&] {
    if (mode != FL_NDCT_LITERAL && mode != FL_NDCT_FAST)
      fail(FL_INVALID_ARGUMENT, "fastleg: unknown ndct mode");
    g_free_mode = mode;
  });
}

int fl_free_ndct_mode(void) { return g_free_mode.load(); }

fl_status fl_nodes_weights(size_t n, double* theta, double* x, double* weights, void* stream) {
  return guarded([&] {
    if (n == 0) fail(FL_INVALID_ARGUMENT, "legendre_nodes_weights: size must be positive");
    require_device();
    cudaStream_t s = as_stream(stream);
    DevOut t(theta, n, 1, n, s), xo(x, n, 1, n, s), wo(weights, n, 1, n, s);
    launch_nodes(n, t.ptr, xo.ptr, wo.ptr, s);
    t.finish();
    xo.finish();
    wo.finish();
    sync(s);
  });
}

fl_status fl_reference_grid(size_t n, int kind, const double* theta, double* theta_star,
                            double* delta_theta, void* stream) {
  return guarded([&] {
    check_kind(kind);
    if (n == 0) return;
    require_device();
    cudaStream_t s = as_stream(stream);
    DevIn th(theta, n, 1, n, s);
    DevOut ts(theta_star, n, 1, n, s), dl(delta_theta, n, 1, n, s);
    launch_reference_grid(n, kind, th.ptr, ts.ptr, dl.ptr, s);
    ts.finish();
    dl.finish();
    sync(s);
  });
}

fl_status fl_lambda_table(size_t max_index, double* table, void* stream) {
  return guarded([&] {
    require_device();
    cudaStream_t s = as_stream(stream);
    DevOut t(table, max_index + 1, 1, max_index + 1, s);
    launch_lambda(max_index, t.ptr, s);
    t.finish();
    sync(s);
  });
}

fl_status fl_trig(int op, int kind, size_t n, const double* in, double* out, size_t batch,
                  size_t ld, void* stream) {
  return guarded([&] {
    if (op < FL_DCT_III || op > FL_DST_III_T) fail(FL_INVALID_ARGUMENT, "fastleg: unknown trig op");
    if (n == 0) fail(FL_INVALID_ARGUMENT, std::string(trig_name(op)) + ": empty input");
    check_kind(kind);
    if (batch == 0) return;
    if (batch == 1) ld = n;
    check_ld(n, ld, batch);
    require_device();
    cudaStream_t s = as_stream(stream);
    DevIn i(in, n, batch, ld, s);
    DevOut o(out, n, batch, ld, s);
    if (i.ld != o.ld) fail(FL_RUNTIME_ERROR, "fastleg: host/device stride mix unsupported");
    if (fast_trig_ok(n, kind))
      fast_trig(op, n, i.ptr, o.ptr, batch, o.ld, s);
    else if (g_free_mode == FL_NDCT_FAST && fast_trig_bessel_ok(n, kind))
      fast_trig_bessel(op, n, i.ptr, o.ptr, batch, o.ld, s);
    else
      czt_trig(op, kind, n, i.ptr, o.ptr, batch, o.ld, s);
    o.finish();
    sync(s);
  });
}

fl_status fl_ndct(int transpose, int kind, size_t n, int num_terms, const double* delta_theta,
                  const double* in, double* out, size_t batch, size_t ld, void* stream) {
  return guarded([&] {
    check_kind(kind);
    const char* where = transpose ? "ndct_apply_transpose" : "ndct_apply";
    if (n == 0 || batch == 0) {
      if (overflow_guard(n, num_terms)) fail(FL_OVERFLOW_ERROR, std::string(where) + ": n^l exceeds double range");
      return;
    }
    if (batch == 1) ld = n;
    check_ld(n, ld, batch);
    require_device();
    cudaStream_t s = as_stream(stream);
    DevIn d(delta_theta, n, 1, n, s);
    DevIn i(in, n, batch, ld, s);
    DevOut o(out, n, batch, ld, s);
    if (i.ld != o.ld) fail(FL_RUNTIME_ERROR, "fastleg: host/device stride mix unsupported");
    const FastNdct* fast = nullptr;
    FastNdctHolder holder;
    // fast mode: the Chebyshev expansion about cheb1 (either kind, power of
    // two) when the literal evaluation is exact to rounding; else literal
    if (num_terms > 0 && g_free_mode == FL_NDCT_FAST && !overflow_guard(n, num_terms))
      holder.p = fast_ndct_create_bessel(n, kind, d.ptr, num_terms, 0, s);
    if (!holder.p && num_terms > 0 && fast_ndct_literal_ok(n, kind))
      holder.p = fast_ndct_create_literal(n, kind, num_terms, d.ptr, s);
    fast = holder.p;
    run_ndct(where, transpose, kind, n, num_terms, d.ptr, i.ptr, i.ld, o.ptr, o.ld, batch,
             nullptr, fast, s);
    o.finish();
    sync(s);
  });
}

fl_status fl_ndct_error_bound(size_t n, int kind, int num_terms, const double* delta_theta,
                              size_t delta_len, const double* coeffs, size_t coeffs_len,
                              double* bound, void* stream) {
  return guarded([&] {
    check_kind(kind);
    // each reduction over its own vector's length, as the reference loops
    // (ndct.hpp:149, :154 norm_l1(coeffs)); q uses the plan size n
    double maxd = 0.0, l1 = 0.0;
    if (delta_len > 0 || coeffs_len > 0) {
      require_device();
      cudaStream_t s = as_stream(stream);
      DevIn d(delta_theta, delta_len, 1, delta_len, s);
      DevIn c(coeffs, coeffs_len, 1, coeffs_len, s);
      DevScratch<double> r(2, s);
      reduce_maxabs_l1(d.ptr, delta_len, c.ptr, coeffs_len, r.p, s);
      double h[2];
      FLB_CUDA(cudaMemcpyAsync(h, r.p, sizeof h, cudaMemcpyDeviceToHost, s));
      sync(s);
      maxd = h[0];
      l1 = h[1];
    }
    // ndct.hpp:150-154
    const double q = static_cast<double>(n) * maxd;
    double node_bound = 1.0;
    for (int l = 1; l <= num_terms; ++l) node_bound *= q / static_cast<double>(l);
    const double qq = kind == FL_CHEB1 ? 0.83845 : 1.0 / (6.0 * kPi);
    double grid_bound = 1.0;
    for (int l = 1; l <= num_terms; ++l) grid_bound *= qq / static_cast<double>(l);
    *bound = (grid_bound < node_bound ? grid_bound : node_bound) * l1;
  });
}

fl_status fl_leg2cheb(int transpose, size_t n, const double* lambda_table, size_t lambda_len,
                      const double* in, double* out, size_t batch, size_t ld, void* stream) {
  return guarded([&] {
    if (n > 0 && lambda_len < n)  // conversion.hpp:90
      fail(FL_INVALID_ARGUMENT, "leg2cheb: Lambda cache smaller than the coefficient vector");
    if (n == 0 || batch == 0) return;
    if (batch == 1) ld = n;
    check_ld(n, ld, batch);
    require_device();
    cudaStream_t s = as_stream(stream);
    DevIn t(lambda_table, n, 1, n, s);
    DevScratch<double> sc(n, s);
    scaled_lambda(t.ptr, sc.p, n, s);
    DevIn i(in, n, batch, ld, s);
    DevOut o(out, n, batch, ld, s);
    if (i.ld != o.ld) fail(FL_RUNTIME_ERROR, "fastleg: host/device stride mix unsupported");
    if (i.ptr == o.ptr) fail(FL_INVALID_ARGUMENT, "leg2cheb: input and output must not alias");
    if (l2c_asy_supported(n) && n >= kL2CAsyMinFree && batch <= kL2CFastMaxCols) {
      // large power-of-two vectors: the asymptotic expansion (tables from this Lambda table)
      L2CAsy* f = l2c_asy_create(n, sc.p, s);
      l2c_asy_one_shot(f);
      try {
        l2c_asy_apply(*f, transpose, i.ptr, o.ptr, batch, o.ld, 0, s);
      } catch (...) {
        FLB_CUDA(cudaStreamSynchronize(s));
        l2c_asy_destroy(f);
        throw;
      }
      FLB_CUDA(cudaStreamSynchronize(s));
      l2c_asy_destroy(f);
    } else if (n >= (size_t(1) << 17) && batch <= kL2CFastMaxCols) {
      // large single vectors: build the low-rank factors for this table once
      L2CFast* f = l2c_fast_create(n, sc.p, s);
      try {
        l2c_fast_apply(*f, transpose, i.ptr, o.ptr, batch, o.ld, 0, s);
      } catch (...) {
        l2c_fast_destroy(f);
        throw;
      }
      FLB_CUDA(cudaStreamSynchronize(s));
      l2c_fast_destroy(f);
    } else {
      leg2cheb_direct(transpose, n, sc.p, i.ptr, o.ptr, batch, o.ld, 0, s);
    }
    o.finish();
    sync(s);
  });
}

fl_status fl_plan_create(size_t n, double tolerance, int kind, fl_plan** plan) {
  return guarded([&] {
    *plan = nullptr;
    // transforms.hpp:21-24 member order: grid, then plan, then Lambda cache
    if (n == 0) fail(FL_INVALID_ARGUMENT, "legendre_nodes_weights: size must be positive");
    check_kind(kind);
    require_device();
    const int L = min_taylor_terms(kind, tolerance);
    fl_plan* p = new fl_plan;
    try {
      p->n = n;
      p->tolerance = tolerance;
      p->kind = kind;
      p->num_terms = L;
      FLB_CUDA(cudaGetDevice(&p->device));
      FLB_CUDA(cudaMalloc(&p->theta, n * 8));
      FLB_CUDA(cudaMalloc(&p->x, n * 8));
      FLB_CUDA(cudaMalloc(&p->w, n * 8));
      launch_nodes(n, p->theta, p->x, p->w, 0);
      plan_finish(p);
    } catch (...) {
      plan_free(p);
      throw;
    }
    *plan = p;
  });
}

fl_status fl_plan_create_from_grid(size_t n, double tolerance, int kind, const double* theta,
                                   const double* x, const double* weights, fl_plan** plan) {
  return guarded([&] {
    *plan = nullptr;
    if (n == 0) fail(FL_INVALID_ARGUMENT, "plan: size must be positive");
    check_kind(kind);
    require_device();
    const int L = min_taylor_terms(kind, tolerance);
    fl_plan* p = new fl_plan;
    try {
      p->n = n;
      p->tolerance = tolerance;
      p->kind = kind;
      p->num_terms = L;
      FLB_CUDA(cudaGetDevice(&p->device));
      FLB_CUDA(cudaMalloc(&p->theta, n * 8));
      FLB_CUDA(cudaMalloc(&p->x, n * 8));
      FLB_CUDA(cudaMalloc(&p->w, n * 8));
      FLB_CUDA(cudaMemcpy(p->theta, theta, n * 8, cudaMemcpyDefault));
      FLB_CUDA(cudaMemcpy(p->x, x, n * 8, cudaMemcpyDefault));
      FLB_CUDA(cudaMemcpy(p->w, weights, n * 8, cudaMemcpyDefault));
      plan_finish(p);
    } catch (...) {
      plan_free(p);
      throw;
    }
    *plan = p;
  });
}

fl_status fl_plan_destroy(fl_plan* plan) {
  return guarded([&] {
    if (plan) plan_free(plan);
  });
}

size_t fl_plan_size(const fl_plan* p) { return p ? p->n : 0; }
int fl_plan_kind(const fl_plan* p) { return p ? p->kind : -1; }
double fl_plan_tolerance(const fl_plan* p) { return p ? p->tolerance : 0.0; }
int fl_plan_num_terms(const fl_plan* p) { return p ? p->num_terms : 0; }

fl_status fl_plan_grid(const fl_plan* p, double* theta, double* x, double* weights) {
  return guarded([&] {
    const size_t b = p->n * 8;
    if (theta) FLB_CUDA(cudaMemcpy(theta, p->theta, b, cudaMemcpyDefault));
    if (x) FLB_CUDA(cudaMemcpy(x, p->x, b, cudaMemcpyDefault));
    if (weights) FLB_CUDA(cudaMemcpy(weights, p->w, b, cudaMemcpyDefault));
  });
}

fl_status fl_plan_reference(const fl_plan* p, double* theta_star, double* delta_theta) {
  return guarded([&] {
    const size_t b = p->n * 8;
    if (theta_star) FLB_CUDA(cudaMemcpy(theta_star, p->tstar, b, cudaMemcpyDefault));
    if (delta_theta) FLB_CUDA(cudaMemcpy(delta_theta, p->delta, b, cudaMemcpyDefault));
  });
}

fl_status fl_plan_lambda(const fl_plan* p, double* table) {
  return guarded([&] { FLB_CUDA(cudaMemcpy(table, p->lambda, p->n * 8, cudaMemcpyDefault)); });
}

fl_status fl_plan_set_ndct_mode(fl_plan* p, int mode) {
  return guarded([&] {
    if (mode != FL_NDCT_LITERAL && mode != FL_NDCT_FAST)
      fail(FL_INVALID_ARGUMENT, "plan: unknown NDCT mode");
    p->mode = mode;
  });
}

int fl_plan_ndct_mode(const fl_plan* p) { return p ? p->mode : -1; }

fl_status fl_plan_ndct(const fl_plan* p, int transpose, const double* in, double* out,
                       size_t batch, size_t ld, void* stream) {
  return guarded([&] {
    if (!p) fail(FL_INVALID_ARGUMENT, "plan: null");
    const size_t n = p->n;
    if (batch == 0) return;
    if (batch == 1) ld = n;
    check_ld(n, ld, batch);
    FLB_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = as_stream(stream);
    DevIn i(in, n, batch, ld, s);
    DevOut o(out, n, batch, ld, s);
    if (i.ld != o.ld) fail(FL_RUNTIME_ERROR, "fastleg: host/device stride mix unsupported");
    const FastNdct* fast = (p->mode == FL_NDCT_FAST) ? p->fast : nullptr;
    run_ndct(transpose ? "ndct_apply_transpose" : "ndct_apply", transpose ? 1 : 0, p->kind, n,
             p->num_terms, p->delta, i.ptr, i.ld, o.ptr, o.ld, batch, nullptr, fast, s);
    o.finish();
    sync(s);
  });
}

int fl_plan_ndct_terms(const fl_plan* p) {
  if (!p) return -1;
  if (p->mode == FL_NDCT_FAST && p->fast) return fast_ndct_dlt_terms(*p->fast);
  return p->num_terms;
}

fl_status fl_plan_stage_terms(const fl_plan* p, int stage, int* count) {
  return guarded([&] {
    *count = 0;
    if (stage == FL_STAGE_LEG2CHEB) {
      if (plan_wants_asy(p, 1)) {
        FLB_CUDA(cudaSetDevice(p->device));
        *count = l2c_asy_terms(*plan_asy(const_cast<fl_plan*>(p), 0));
        return;
      }
      FLB_CUDA(cudaSetDevice(p->device));
      const L2CFast* th = plan_th(p, 0);
      if (!th) fail(FL_INVALID_ARGUMENT, "dlt_stage: no Toeplitz-Hankel conversion for this size");
      *count = std::max(l2c_fast_rank(*th, 0), l2c_fast_rank(*th, 1));
    } else if (stage == FL_STAGE_NDCT) {
      if (!p->fast || p->n <= 8192)
        fail(FL_INVALID_ARGUMENT, "dlt_stage: term-parallel NDCT needs a power-of-two N > 8192");
      *count = fast_ndct_terms(*p->fast);
    } else {
      fail(FL_INVALID_ARGUMENT, "dlt_stage: unknown stage");
    }
  });
}

fl_status fl_plan_stage_cost(const fl_plan* p, int stage, int term, double* cost) {
  return guarded([&] {
    int count = 0;
    const fl_status st = fl_plan_stage_terms(p, stage, &count);
    if (st != FL_OK) fail(st, fl_last_error());
    if (term < 0 || term >= count) fail(FL_INVALID_ARGUMENT, "dlt_stage: term out of bounds");
    *cost = stage == FL_STAGE_LEG2CHEB && plan_wants_asy(p, 1)
                ? l2c_asy_term_cost(*plan_asy(const_cast<fl_plan*>(p), 0), term)
                : 1.0;
  });
}

fl_status fl_dlt_stage(const fl_plan* p, int inverse, int stage, int lo, int hi, const double* in,
                       double* out, void* stream) {
  return guarded([&] {
    int count = 0;
    const fl_status st = fl_plan_stage_terms(p, stage, &count);
    if (st != FL_OK) fail(st, fl_last_error());
    if (lo < 0 || hi > count || lo > hi) fail(FL_INVALID_ARGUMENT, "dlt_stage: term range out of bounds");
    const size_t n = p->n;
    FLB_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = as_stream(stream);
    DevIn i(in, n, 1, n, s);
    DevOut o(out, n, 1, n, s);
    if (lo == hi) {
      FLB_CUDA(cudaMemsetAsync(o.ptr, 0, n * sizeof(double), s));
    } else if (stage == FL_STAGE_LEG2CHEB) {
      if (plan_wants_asy(p, 1))
        l2c_asy_apply(*plan_asy(const_cast<fl_plan*>(p), s), inverse, i.ptr, o.ptr, 1, n, inverse, s, lo,
                      hi);
      else
        l2c_fast_apply(*plan_th(p, s), inverse, i.ptr, o.ptr, 1, n, inverse, s, lo, hi);
    } else {
      SyncFlag flag;
      fast_ndct_run(*p->fast, inverse, i.ptr, n, o.ptr, n, 1, inverse ? p->w : nullptr, flag.p, s,
                    lo, hi);
      const bool h = flag.wait(s);
      if (h) fail(FL_INVALID_ARGUMENT, inverse ? "ndct_apply_transpose: non-finite input"
                                               : "ndct_apply: non-finite input");
    }
    o.finish();
    sync(s);
  });
}

struct fl_fs {
  const fl_plan* plan = nullptr;
  FsLayout* lay = nullptr;
  int* flag = nullptr;  // non-finite input seen by a part-1 call
};

fl_status fl_fs_create(const fl_plan* p, int world, int rank, fl_fs** out) {
  return guarded([&] {
    if (!p || !out) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    *out = nullptr;
    if (!p->fast || p->mode != FL_NDCT_FAST)
      fail(FL_INVALID_ARGUMENT, "four-step: needs a fast-mode plan of power-of-two size");
    FLB_CUDA(cudaSetDevice(p->device));
    auto* f = new fl_fs;
    f->plan = p;
    try {
      f->lay = fs_create(p->n, world, rank);
      FLB_CUDA(cudaMalloc(&f->flag, sizeof(int)));
      FLB_CUDA(cudaMemset(f->flag, 0, sizeof(int)));
    } catch (...) {
      if (f->lay) fs_destroy(f->lay);
      if (f->flag) cudaFree(f->flag);
      delete f;
      throw;
    }
    *out = f;
  });
}

fl_status fl_fs_destroy(fl_fs* f) {
  return guarded([&] {
    if (!f) return;
    fs_destroy(f->lay);
    if (f->flag) cudaFree(f->flag);
    delete f;
  });
}

fl_status fl_fs_info(const fl_fs* f, size_t* info) {
  return guarded([&] {
    if (!f || !info) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    const FsInfo i = fs_info(*f->lay);
    const size_t v[10] = {i.n, i.L, i.L1, i.L2, i.KB, i.B, i.nres, i.res_max, (size_t)i.world,
                          (size_t)i.rank};
    std::copy(v, v + 10, info);
  });
}

fl_status fl_fs_coef_count(const fl_fs* f, int transpose, int peer, int send, size_t* count) {
  return guarded([&] {
    if (!f || !count) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    *count = fs_coef_count(*f->lay, transpose, peer, send);
  });
}

size_t fl_fs_work_elems(const fl_fs* f, int terms) {
  if (!f || terms <= 0) return 0;
  const FsInfo i = fs_info(*f->lay);
  // rows of either FFT stage: terms x max(nres L2, KB L1)
  return (size_t)terms * std::max(i.nres * i.L2, i.KB * i.L1);
}

fl_status fl_fs_to_residue(const fl_fs* f, const double* full, double* slabs, void* stream) {
  return guarded([&] {
    if (!f || !full || !slabs) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    FLB_CUDA(cudaSetDevice(f->plan->device));
    fs_to_residue(*f->lay, full, slabs, as_stream(stream));
  });
}

fl_status fl_fs_from_residue(const fl_fs* f, const double* slabs, double* full, void* stream) {
  return guarded([&] {
    if (!f || !full || !slabs) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    FLB_CUDA(cudaSetDevice(f->plan->device));
    fs_from_residue(*f->lay, slabs, full, as_stream(stream));
  });
}

fl_status fl_fs_values(const fl_fs* f, int to_block, const double* in, double* out, void* stream) {
  return guarded([&] {
    if (!f || !in || !out) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    FLB_CUDA(cudaSetDevice(f->plan->device));
    if (to_block)
      fs_values_from_exchange(*f->lay, in, out, as_stream(stream));
    else
      fs_values_to_exchange(*f->lay, in, out, as_stream(stream));
  });
}

fl_status fl_fs_ndct_part(const fl_fs* f, int transpose, int part, int t0, int t1, const void* in,
                          void* out, void* work, int first, void* stream) {
  return guarded([&] {
    if (!f || !in || !out || !work) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    const fl_plan* p = f->plan;
    FLB_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = as_stream(stream);
    auto* w = static_cast<double2*>(work);
    if (part == 1 && !transpose)
      fs_fwd1(*f->lay, *p->fast, t0, t1, static_cast<const double*>(in), static_cast<double2*>(out), w,
              f->flag, s);
    else if (part == 2 && !transpose)
      fs_fwd2(*f->lay, *p->fast, t0, t1, static_cast<const double2*>(in), w, static_cast<double*>(out),
              first, s);
    else if (part == 1)
      fs_tr1(*f->lay, *p->fast, p->w, t0, t1, static_cast<const double*>(in), static_cast<double2*>(out),
             w, f->flag, s);
    else if (part == 2)
      fs_tr2(*f->lay, *p->fast, t0, t1, static_cast<const double2*>(in), w, static_cast<double*>(out),
             first, s);
    else
      fail(FL_INVALID_ARGUMENT, "four-step: part must be 1 or 2");
  });
}

fl_status fl_fs_check(const fl_fs* f, int transpose, void* stream) {
  return guarded([&] {
    if (!f) fail(FL_INVALID_ARGUMENT, "four-step: null argument");
    FLB_CUDA(cudaSetDevice(f->plan->device));
    cudaStream_t s = as_stream(stream);
    int h = 0;
    FLB_CUDA(cudaMemcpyAsync(&h, f->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync(s);
    if (h) {
      FLB_CUDA(cudaMemset(f->flag, 0, sizeof(int)));
      fail(FL_INVALID_ARGUMENT, transpose ? "ndct_apply_transpose: non-finite input"
                                          : "ndct_apply: non-finite input");
    }
  });
}

fl_status fl_plan_set_leg2cheb_mode(fl_plan* p, int mode) {
  return guarded([&] {
    if (mode != FL_LEG2CHEB_DIRECT && mode != FL_LEG2CHEB_FAST && mode != FL_LEG2CHEB_ASYMPTOTIC &&
        mode != FL_LEG2CHEB_TOEPLITZ)
      fail(FL_INVALID_ARGUMENT, "plan: unknown leg2cheb mode");
    p->l2c_mode = mode;
  });
}

fl_status fl_plan_leg2cheb_asy_info(const fl_plan* p, int* terms, int* levels, int* transforms,
                                    double* steps) {
  return guarded([&] {
    if (!p) fail(FL_INVALID_ARGUMENT, "plan: null");
    FLB_CUDA(cudaSetDevice(p->device));
    const L2CAsy* a = plan_asy(const_cast<fl_plan*>(p), 0);
    if (!a) fail(FL_INVALID_ARGUMENT, "leg2cheb: no asymptotic conversion for this size");
    const L2CAsyInfo i = l2c_asy_info(*a);
    if (terms) *terms = i.M;
    if (levels) *levels = i.levels;
    if (transforms) *transforms = i.transforms;
    if (steps) *steps = i.rec_steps_per_n;
  });
}

fl_status fl_plan_leg2cheb(const fl_plan* p, int transpose, const double* in, double* out,
                           size_t batch, size_t ld, void* stream) {
  return guarded([&] {
    if (!p) fail(FL_INVALID_ARGUMENT, "plan: null");
    const size_t n = p->n;
    if (batch == 0) return;
    if (batch == 1) ld = n;
    check_ld(n, ld, batch);
    FLB_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = as_stream(stream);
    DevIn i(in, n, batch, ld, s);
    DevOut o(out, n, batch, ld, s);
    const double* cin = i.ptr;
    DevScratch<double> packed(i.ld != n ? n * batch : 0, s);
    if (i.ld != n) {
      FLB_CUDA(cudaMemcpy2DAsync(packed.p, n * 8, i.ptr, i.ld * 8, n * 8, batch,
                                 cudaMemcpyDeviceToDevice, s));
      cin = packed.p;
    }
    plan_convert(const_cast<fl_plan*>(p), transpose ? 1 : 0, cin, o.ptr, batch, o.ld, s);
    o.finish();
    sync(s);
  });
}

fl_status fl_plan_set_gemm_mode(fl_plan* p, int mode) {
  return guarded([&] {
    if (!p) fail(FL_INVALID_ARGUMENT, "plan: null");
    if (mode != FL_GEMM_FP64 && mode != FL_GEMM_INT8_SPLIT)
      fail(FL_INVALID_ARGUMENT, "plan: unknown gemm mode");
    p->gemm_mode = mode;
  });
}

int fl_plan_gemm_mode(const fl_plan* p) { return p ? p->gemm_mode : -1; }

fl_status fl_plan_set_dlt_method(fl_plan* p, int method) {
  return guarded([&] {
    if (!p) fail(FL_INVALID_ARGUMENT, "plan: null");
    if (method != FL_DLT_FACTORED && method != FL_DLT_DIRECT)
      fail(FL_INVALID_ARGUMENT, "plan: unknown dlt method");
    p->dlt_method = method;
  });
}

int fl_plan_dlt_method(const fl_plan* p) { return p ? p->dlt_method : -1; }

int fl_plan_uses_direct(const fl_plan* p, size_t batch) {
  return p && p->dlt_method == FL_DLT_DIRECT && p->gemm_mode == FL_GEMM_INT8_SPLIT && batch > 16 &&
                 l2c_dense_supported(p->n)
             ? 1
             : 0;
}

int fl_plan_leg2cheb_rank(const fl_plan* p, int parity) {
  if (!p || parity < 0 || parity > 1) return 0;
  // builds the factors on first query (0 below 2^14, or when they fail)
  L2CFast* th = nullptr;
  if (guarded([&] {
        FLB_CUDA(cudaSetDevice(p->device));
        th = plan_th(p, 0);
      }) != FL_OK)
    return 0;
  return th ? l2c_fast_rank(*th, parity) : 0;
}

fl_status fl_dlt(const fl_plan* p, const double* in, double* out, size_t batch, size_t ld,
                 void* stream) {
  return guarded([&] {
    const size_t n = p->n;
    if (batch == 0) return;
    if (batch == 1) ld = n;
    check_ld(n, ld, batch);
    FLB_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = as_stream(stream);
    const FastNdct* fast = (p->mode == FL_NDCT_FAST) ? p->fast : nullptr;
    fl_plan* mp = const_cast<fl_plan*>(p);
    // the direct product (P c on the int8 tensor cores) where it applies
    if (const L2COzaki* dense = plan_dense(mp, 0, batch, s)) {
      if (pipeline_ok(in, out, n, batch)) {
        run_pipelined(p->device, n, in, out, batch, ld, s, "ndct_apply",
                      [&](const double* di, double* dq, size_t cols, int* flag, cudaStream_t cs) {
                        l2c_dense_apply(*dense, di, n, nullptr, dq, n, cols, flag, cs);
                      });
        return;
      }
      DevIn i(in, n, batch, ld, s);
      DevOut o(out, n, batch, ld, s);
      SyncFlag flag;
      l2c_dense_apply(*dense, i.ptr, i.ld, nullptr, o.ptr, o.ld, batch, flag.p, s);
      o.finish();
      const bool h = flag.wait(s);
      // the reference raises on the non-finite conversion output (ndct.hpp:79-91)
      if (h) fail(FL_INVALID_ARGUMENT, "ndct_apply: non-finite input");
      return;
    }
    if (const DenseGemv* g = plan_gemv(mp, batch, s)) {
      DevIn i(in, n, batch, ld, s);
      DevOut o(out, n, batch, ld, s);
      SyncFlag flag;
      dense_gemv_dlt(*g, i.ptr, i.ld, o.ptr, o.ld, batch, flag.p, s);
      o.finish();
      const bool h = flag.wait(s);
      if (h) fail(FL_INVALID_ARGUMENT, "ndct_apply: non-finite input");
      return;
    }
    if (pipeline_ok(in, out, n, batch) && !overflow_guard(n, p->num_terms)) {
      run_pipelined(p->device, n, in, out, batch, ld, s, "ndct_apply",
                    [&](const double* di, double* dq, size_t cols, int* flag, cudaStream_t cs) {
                      DevScratch<double> chat(n * cols, cs);
                      plan_convert(mp, 0, di, chat.p, cols, n, cs);
                      enqueue_ndct(0, p->kind, n, p->num_terms, p->delta, chat.p, n, dq, n, cols,
                                   nullptr, fast, flag, cs);
                    });
      return;
    }
    DevIn i(in, n, batch, ld, s);
    DevOut o(out, n, batch, ld, s);
    if (i.ld != o.ld) fail(FL_RUNTIME_ERROR, "fastleg: host/device stride mix unsupported");
    // transforms.hpp:47-48: chat = M c (scratch), f = NDCT(chat)
    DevScratch<double> chat(n * batch, s);
    const double* cin = i.ptr;
    DevScratch<double> packed(i.ld != n ? n * batch : 0, s);
    if (i.ld != n) {  // the conversion kernels read columns of stride n
      FLB_CUDA(cudaMemcpy2DAsync(packed.p, n * 8, i.ptr, i.ld * 8, n * 8, batch,
                                 cudaMemcpyDeviceToDevice, s));
      cin = packed.p;
    }
    plan_convert(mp, 0, cin, chat.p, batch, n, s);
    DeferredNdct nd(s);
    if (o.ld != n) {
      DevScratch<double> f(n * batch, s);
      nd.run("ndct_apply", 0, p->kind, n, p->num_terms, p->delta, chat.p, n, f.p, n, batch,
             nullptr, fast, s);
      FLB_CUDA(cudaMemcpy2DAsync(o.ptr, o.ld * 8, f.p, n * 8, n * 8, batch,
                                 cudaMemcpyDeviceToDevice, s));
    } else {
      nd.run("ndct_apply", 0, p->kind, n, p->num_terms, p->delta, chat.p, n, o.ptr, n, batch,
             nullptr, fast, s);
    }
    o.finish();
    nd.finish(s);
  });
}

fl_status fl_idlt(const fl_plan* p, const double* in, double* out, size_t batch, size_t ld,
                  void* stream) {
  return guarded([&] {
    const size_t n = p->n;
    if (batch == 0) return;
    if (batch == 1) ld = n;
    check_ld(n, ld, batch);
    FLB_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = as_stream(stream);
    const FastNdct* fast = (p->mode == FL_NDCT_FAST) ? p->fast : nullptr;
    fl_plan* mp = const_cast<fl_plan*>(p);
    if (const L2COzaki* dense = plan_dense(mp, 1, batch, s)) {
      if (pipeline_ok(in, out, n, batch)) {
        run_pipelined(p->device, n, in, out, batch, ld, s, "ndct_apply_transpose",
                      [&](const double* di, double* dq, size_t cols, int* flag, cudaStream_t cs) {
                        l2c_dense_apply(*dense, di, n, p->w, dq, n, cols, flag, cs);
                      });
        return;
      }
      DevIn i(in, n, batch, ld, s);
      DevOut o(out, n, batch, ld, s);
      SyncFlag flag;
      l2c_dense_apply(*dense, i.ptr, i.ld, p->w, o.ptr, o.ld, batch, flag.p, s);
      o.finish();
      const bool h = flag.wait(s);
      if (h) fail(FL_INVALID_ARGUMENT, "ndct_apply_transpose: non-finite input");
      return;
    }
    if (const DenseGemv* g = plan_gemv(mp, batch, s)) {
      DevIn i(in, n, batch, ld, s);
      DevOut o(out, n, batch, ld, s);
      SyncFlag flag;
      dense_gemv_idlt(*g, i.ptr, i.ld, p->w, o.ptr, o.ld, batch, flag.p, s);
      o.finish();
      const bool h = flag.wait(s);
      if (h) fail(FL_INVALID_ARGUMENT, "ndct_apply_transpose: non-finite input");
      return;
    }
    if (pipeline_ok(in, out, n, batch) && !overflow_guard(n, p->num_terms)) {
      run_pipelined(p->device, n, in, out, batch, ld, s, "ndct_apply_transpose",
                    [&](const double* di, double* dq, size_t cols, int* flag, cudaStream_t cs) {
                      DevScratch<double> back(n * cols, cs);
                      enqueue_ndct(1, p->kind, n, p->num_terms, p->delta, di, n, back.p, n, cols,
                                   p->w, fast, flag, cs);
                      plan_convert(mp, 1, back.p, dq, cols, n, cs);
                    });
      return;
    }
    DevIn i(in, n, batch, ld, s);
    DevOut o(out, n, batch, ld, s);
    // transforms.hpp:58-62: back = NDCT^T(w . f); c = (m + 1/2) M^T back
    DevScratch<double> back(n * batch, s);
    DeferredNdct nd(s);
    if (i.ld != n) {
      DevScratch<double> f(n * batch, s);
      FLB_CUDA(cudaMemcpy2DAsync(f.p, n * 8, i.ptr, i.ld * 8, n * 8, batch,
                                 cudaMemcpyDeviceToDevice, s));
      nd.run("ndct_apply_transpose", 1, p->kind, n, p->num_terms, p->delta, f.p, n, back.p, n,
             batch, p->w, fast, s);
    } else {
      nd.run("ndct_apply_transpose", 1, p->kind, n, p->num_terms, p->delta, i.ptr, n, back.p, n,
             batch, p->w, fast, s);
    }
    plan_convert(mp, 1, back.p, o.ptr, batch, o.ld, s);
    o.finish();
    nd.finish(s);
  });
}

static fl_status direct_eval_entry(int chebyshev, const double* c, size_t n, const double* xs,
                                   size_t m, double* out, void* stream) {
  return guarded([&] {
    if (m == 0) return;
    require_device();
    cudaStream_t s = as_stream(stream);
    DevIn x(xs, m, 1, m, s);
    if (!direct_domain_ok(x.ptr, m, s))
      fail(FL_DOMAIN_ERROR, std::string(chebyshev ? "eval_chebyshev_direct" : "eval_legendre_direct") +
                                ": abscissa outside [-1, 1]");
    DevIn cc(c, n, 1, n, s);
    DevOut o(out, m, 1, m, s);
    direct_eval(chebyshev, cc.ptr, n, x.ptr, m, o.ptr, s);
    o.finish();
    sync(s);
  });
}

fl_status fl_eval_legendre_direct(const double* c, size_t n, const double* xs, size_t m,
                                  double* out, void* stream) {
  return direct_eval_entry(0, c, n, xs, m, out, stream);
}

fl_status fl_eval_chebyshev_direct(const double* c, size_t n, const double* xs, size_t m,
                                   double* out, void* stream) {
  return direct_eval_entry(1, c, n, xs, m, out, stream);
}

fl_status fl_idlt_direct(const double* f, size_t n, const double* x, const double* weights,
                         double* out, void* stream) {
  return guarded([&] {
    if (n == 0) return;
    require_device();
    cudaStream_t s = as_stream(stream);
    DevIn ff(f, n, 1, n, s), xx(x, n, 1, n, s), ww(weights, n, 1, n, s);
    DevOut o(out, n, 1, n, s);
    direct_idlt(ff.ptr, xx.ptr, ww.ptr, n, o.ptr, s);
    o.finish();
    sync(s);
  });
}

fl_status fl_cheb_coeffs_of_legendre(size_t n, size_t m, double* out, void* stream) {
  return guarded([&] {
    if (m <= n)
      fail(FL_INVALID_ARGUMENT, "cheb_coeffs_of_legendre: need more sample points than degree");
    require_device();
    cudaStream_t s = as_stream(stream);
    DevOut o(out, n + 1, 1, n + 1, s);
    direct_cheb_coeffs(n, m, o.ptr, s);
    o.finish();
    sync(s);
  });
}

// random.hpp:15-55 (host input generation; not part of the device path)
static void gen_columns(size_t n, size_t batch, int threads,
                        void (*col)(size_t n, uint64_t seed, double* out, double decay),
                        uint64_t seed, double* out, double decay) {
  if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
  if (threads <= 0) threads = 1;
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (;;) {
      const size_t j = next.fetch_add(1);
      if (j >= batch) break;
      col(n, seed + j, out + j * n, decay);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads && (size_t)t < batch; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
}

static void decaying_column(size_t n, uint64_t seed, double* out, double decay) {
  std::mt19937_64 rng(seed);
  auto u01 = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
  bool have = false;
  double spare = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double g;
    if (have) {
      have = false;
      g = spare;
    } else {
      double u1;
      do {
        u1 = u01();
      } while (u1 == 0.0);
      const double u2 = u01();
      const double r = std::sqrt(-2.0 * std::log(u1));
      have = true;
      spare = r * std::sin(2.0 * kPi * u2);
      g = r * std::cos(2.0 * kPi * u2);
    }
    out[i] = g * std::pow(static_cast<double>(i + 1), -decay);
  }
}

static void uniform_column(size_t n, uint64_t seed, double* out, double) {
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = 2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0;
}

// ---- vector_io.hpp with pinned staging --------------------------------------
namespace {
constexpr size_t kIoChunk = size_t(1) << 20;  // doubles per staged chunk (8 MiB)

struct Pinned {
  double* p = nullptr;
  explicit Pinned(size_t n) { FLB_CUDA(cudaMallocHost(&p, (n ? n : 1) * sizeof(double))); }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

uint64_t le64(const unsigned char* b) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}
}  // namespace

fl_status fl_load_vector(const char* path, int format, double* out, size_t capacity,
                         size_t* count, void* stream) {
  return guarded([&] {
    if (format != 0 && format != 1) fail(FL_INVALID_ARGUMENT, "vector_io: unknown format");
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(FL_RUNTIME_ERROR, std::string("cannot open for reading: ") + path);
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    const bool dev = is_device_ptr(out);
    cudaStream_t s = as_stream(stream);
    if (format == 0) {  // csv: parse on the host (vector_io.hpp:66-80), one staged copy
      std::vector<double> vals;
      char line[512];
      for (size_t lineno = 1; std::fgets(line, sizeof line, f); ++lineno) {
        char* b = line;
        while (*b == ' ' || *b == '\t' || *b == '\r') ++b;
        char* e = b + std::strlen(b);
        while (e > b && (e[-1] == ' ' || e[-1] == '\t' || e[-1] == '\r' || e[-1] == '\n')) --e;
        if (e == b) continue;
        *e = '\0';
        char* end = nullptr;
        const double v = std::strtod(b, &end);
        if (end != e)
          fail(FL_RUNTIME_ERROR, std::string(path) + ":" + std::to_string(lineno) +
                                     ": not a number: '" + b + "'");
        vals.push_back(v);
      }
      *count = vals.size();
      if (vals.size() > capacity) fail(FL_INVALID_ARGUMENT, "vector_io: output too small");
      if (vals.empty()) return;
      if (!dev) {
        std::memcpy(out, vals.data(), vals.size() * 8);
        return;
      }
      Pinned st(vals.size());
      std::memcpy(st.p, vals.data(), vals.size() * 8);
      FLB_CUDA(cudaMemcpyAsync(out, st.p, vals.size() * 8, cudaMemcpyHostToDevice, s));
      sync(s);
      return;
    }
    unsigned char head[16];
    if (std::fread(head, 1, 8, f) != 8 || std::memcmp(head, "FLEGVEC1", 8) != 0)
      fail(FL_RUNTIME_ERROR, std::string(path) + ": bad magic, not a vector file");
    if (std::fread(head + 8, 1, 8, f) != 8)
      fail(FL_RUNTIME_ERROR, std::string(path) + ": truncated header");
    const uint64_t n = le64(head + 8);
    *count = (size_t)n;
    if (n > capacity) fail(FL_INVALID_ARGUMENT, "vector_io: output too small");
    // two pinned chunks: the H2D copy of one overlaps the read of the next
    // (binary64 LE is the device's layout on x86 hosts: no per-element work)
    const size_t chunk = std::min<size_t>(kIoChunk, n ? n : 1);
    Pinned buf[2] = {Pinned(chunk), Pinned(chunk)};
    cudaEvent_t done[2];
    for (cudaEvent_t& e : done) FLB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    bool used[2] = {false, false};
    size_t i0 = 0;
    int b = 0;
    bool ok = true;
    while (i0 < n) {
      const size_t m = std::min<size_t>(chunk, n - i0);
      if (used[b]) FLB_CUDA(cudaEventSynchronize(done[b]));
      if (std::fread(buf[b].p, 8, m, f) != m) {
        ok = false;
        break;
      }
      if (dev) {
        FLB_CUDA(cudaMemcpyAsync(out + i0, buf[b].p, m * 8, cudaMemcpyHostToDevice, s));
        FLB_CUDA(cudaEventRecord(done[b], s));
        used[b] = true;
      } else {
        std::memcpy(out + i0, buf[b].p, m * 8);
      }
      i0 += m;
      b ^= 1;
    }
    FLB_CUDA(cudaStreamSynchronize(s));
    for (cudaEvent_t e : done) cudaEventDestroy(e);
    if (!ok) fail(FL_RUNTIME_ERROR, std::string(path) + ": truncated payload");
  });
}

fl_status fl_save_vector(const char* path, int format, const double* in, size_t n, void* stream) {
  return guarded([&] {
    if (format != 0 && format != 1) fail(FL_INVALID_ARGUMENT, "vector_io: unknown format");
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(FL_RUNTIME_ERROR, std::string("cannot open for writing: ") + path);
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    const bool dev = is_device_ptr(in);
    cudaStream_t s = as_stream(stream);
    if (format == 1) {
      unsigned char head[16];
      std::memcpy(head, "FLEGVEC1", 8);
      for (int i = 0; i < 8; ++i) head[8 + i] = (unsigned char)((uint64_t)n >> (8 * i));
      if (std::fwrite(head, 1, 16, f) != 16) fail(FL_RUNTIME_ERROR, std::string("write failed: ") + path);
    }
    const size_t chunk = std::min<size_t>(kIoChunk, n ? n : 1);
    Pinned buf[2] = {Pinned(chunk), Pinned(chunk)};
    cudaEvent_t done[2];
    for (cudaEvent_t& e : done) FLB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // D2H of chunk i + 1 runs while chunk i is written
    auto issue = [&](size_t i0, int b) {
      const size_t m = std::min<size_t>(chunk, n - i0);
      if (dev) {
        FLB_CUDA(cudaMemcpyAsync(buf[b].p, in + i0, m * 8, cudaMemcpyDeviceToHost, s));
        FLB_CUDA(cudaEventRecord(done[b], s));
      } else {
        std::memcpy(buf[b].p, in + i0, m * 8);
      }
    };
    bool ok = true;
    if (n) issue(0, 0);
    int b = 0;
    char txt[32];
    for (size_t i0 = 0; i0 < n; i0 += chunk, b ^= 1) {
      const size_t m = std::min<size_t>(chunk, n - i0);
      if (dev) FLB_CUDA(cudaEventSynchronize(done[b]));
      if (i0 + chunk < n) issue(i0 + chunk, b ^ 1);
      if (format == 1) {
        ok = ok && std::fwrite(buf[b].p, 8, m, f) == m;
      } else {
        for (size_t i = 0; i < m; ++i) {  // shortest round-trip decimal (vector_io.hpp:56-60)
          const auto r = std::to_chars(txt, txt + sizeof txt, buf[b].p[i]);
          *r.ptr = '\n';
          ok = ok && std::fwrite(txt, 1, (size_t)(r.ptr + 1 - txt), f) == (size_t)(r.ptr + 1 - txt);
        }
      }
    }
    FLB_CUDA(cudaStreamSynchronize(s));
    for (cudaEvent_t e : done) cudaEventDestroy(e);
    if (!ok || std::fflush(f) != 0) fail(FL_RUNTIME_ERROR, std::string("write failed: ") + path);
  });
}

void fl_random_decaying(size_t n, double decay, uint64_t seed, double* out, size_t batch,
                        int threads) {
  gen_columns(n, batch, threads, decaying_column, seed, out, decay);
}

void fl_random_uniform_pm1(size_t n, uint64_t seed, double* out, size_t batch, int threads) {
  gen_columns(n, batch, threads, uniform_column, seed, out, 0.0);
}

}  // extern "C"
