// Batched power-of-two complex fp64 FFT: shared-memory Stockham for
// P <= 8192, six-step (transpose / row FFTs / twiddle-transpose / row FFTs /
// transpose) through HBM above that.
#include <map>
#include <mutex>
#include <cmath>
#include <utility>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "launch.cuh"

namespace flb {

namespace {

__global__ void twiddle_kernel(double2* tw, unsigned long long p) {
  const unsigned long long m = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (m >= p) return;
  double s, c;
  sincospi(2.0 * (double)m / (double)p, &s, &c);
  tw[m] = make_double2(c, -s);
}

template <int LOG2P, bool INV>
__global__ void __launch_bounds__(512) fft_smem_kernel(double2* __restrict__ data, size_t rows,
                                                       const double2* __restrict__ tw) {
  constexpr int P = 1 << LOG2P;
  constexpr int E = P >= 8192 ? 16 : 8;
  constexpr int TR = P / E;
  constexpr int RPC = TR >= 256 ? 1 : 256 / TR;
  extern __shared__ double2 sm[];
  const size_t row0 = (size_t)blockIdx.x * RPC;
  for (int i = threadIdx.x; i < RPC * P; i += blockDim.x) {
    const size_t r = row0 + i / P;
    sm[(i / P) * smem_row(P) + smem_pad(i % P)] = r < rows ? data[r * P + (i % P)] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int lr = threadIdx.x / TR, tid = threadIdx.x % TR;
  fft_row_smem<P, E, INV>(sm + lr * smem_row(P), tid, tw);
  for (int i = threadIdx.x; i < RPC * P; i += blockDim.x) {
    const size_t r = row0 + i / P;
    if (r < rows) data[r * P + (i % P)] = sm[(i / P) * smem_row(P) + smem_pad(i % P)];
  }
}

// P in {1, 2, 4}: direct DFT, one thread per row
template <bool INV>
__global__ void fft_tiny_kernel(double2* __restrict__ data, size_t rows, int p) {
  const size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double2 v[4], o[4];
  for (int i = 0; i < p; ++i) v[i] = data[r * p + i];
  for (int k = 0; k < p; ++k) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < p; ++j) {
      const int m = (j * k) % p;
      double s, c;
      sincospi(2.0 * (double)m / (double)p, &s, &c);
      if (!INV) s = -s;
      acc.x += v[j].x * c - v[j].y * s;
      acc.y += v[j].x * s + v[j].y * c;
    }
    o[k] = acc;
  }
  for (int i = 0; i < p; ++i) data[r * p + i] = o[i];
}

// out[item][c][r] = in[item][r][c] * (twiddle ? w_P^{r c} : 1)
template <bool INV>
__global__ void transpose_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                 int rows, int cols, unsigned long long twiddle_p) {
  __shared__ double2 tile[32][33];
  const size_t item = blockIdx.z;
  const size_t plane = (size_t)rows * cols;
  const double2* src = in + item * plane;
  double2* dst = out + item * plane;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const int r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = src[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const int c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      double2 v = tile[threadIdx.x][dy];
      if (twiddle_p) {
        const unsigned long long m = ((unsigned long long)r * (unsigned long long)c) % twiddle_p;
        double s, co;
        sincospi(2.0 * (double)m / (double)twiddle_p, &s, &co);
        if (!INV) s = -s;
        v = make_double2(v.x * co - v.y * s, v.x * s + v.y * co);
      }
      dst[(size_t)c * rows + r] = v;
    }
  }
}

template <int LOG2P, bool INV>
void launch_smem(double2* data, size_t rows, const double2* tw, cudaStream_t s) {
  constexpr int P = 1 << LOG2P;
  constexpr int E = P >= 8192 ? 16 : 8;
  constexpr int TR = P / E;
  constexpr int RPC = TR >= 256 ? 1 : 256 / TR;
  const size_t smem = (size_t)RPC * smem_row(P) * sizeof(double2);
  FLB_CUDA(cudaFuncSetAttribute(fft_smem_kernel<LOG2P, INV>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const size_t grid = (rows + RPC - 1) / RPC;
  fft_smem_kernel<LOG2P, INV><<<(unsigned)grid, TR * RPC, smem, s>>>(data, rows, tw);
  note_launch("fft_smem_kernel");
}

template <bool INV>
void launch_smem_dispatch(int log2p, double2* data, size_t rows, const double2* tw,
                          cudaStream_t s) {
  switch (log2p) {
    case 3: launch_smem<3, INV>(data, rows, tw, s); break;
    case 4: launch_smem<4, INV>(data, rows, tw, s); break;
    case 5: launch_smem<5, INV>(data, rows, tw, s); break;
    case 6: launch_smem<6, INV>(data, rows, tw, s); break;
    case 7: launch_smem<7, INV>(data, rows, tw, s); break;
    case 8: launch_smem<8, INV>(data, rows, tw, s); break;
    case 9: launch_smem<9, INV>(data, rows, tw, s); break;
    case 10: launch_smem<10, INV>(data, rows, tw, s); break;
    case 11: launch_smem<11, INV>(data, rows, tw, s); break;
    case 12: launch_smem<12, INV>(data, rows, tw, s); break;
    case 13: launch_smem<13, INV>(data, rows, tw, s); break;
    default: fail(FL_RUNTIME_ERROR, "fft: unsupported shared-memory size");
  }
}

void transpose(const double2* in, double2* out, int rows, int cols, size_t items,
               unsigned long long twiddle_p, bool inverse, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, (unsigned)items);
  if (items > 65535) fail(FL_RUNTIME_ERROR, "fft: too many transforms in one six-step call");
  if (inverse)
    transpose_kernel<true><<<grid, block, 0, s>>>(in, out, rows, cols, twiddle_p);
  else
    transpose_kernel<false><<<grid, block, 0, s>>>(in, out, rows, cols, twiddle_p);
  note_launch("transpose_kernel");
}

void fft_rows(double2* data, int log2p, size_t rows, bool inverse, cudaStream_t s) {
  if (log2p <= 2) {
    const int threads = 128;
    const unsigned grid = (unsigned)((rows + threads - 1) / threads);
    if (inverse)
      fft_tiny_kernel<true><<<grid, threads, 0, s>>>(data, rows, 1 << log2p);
    else
      fft_tiny_kernel<false><<<grid, threads, 0, s>>>(data, rows, 1 << log2p);
    note_launch("fft_tiny_kernel");
    return;
  }
  const double2* tw = pass_twiddles(log2p);
  if (inverse)
    launch_smem_dispatch<true>(log2p, data, rows, tw, s);
  else
    launch_smem_dispatch<false>(log2p, data, rows, tw, s);
}

}  // namespace

const double2* twiddle_table(int log2p) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, double2*> tables;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  double2*& slot = tables[{dev, log2p}];
  if (!slot) {
    const unsigned long long p = 1ull << log2p;
    FLB_CUDA(cudaMalloc(&slot, p * sizeof(double2)));
    twiddle_kernel<<<(unsigned)((p + 255) / 256), 256>>>(slot, p);
    note_launch("twiddle_kernel");
    FLB_CUDA(cudaDeviceSynchronize());
  }
  return slot;
}

const double2* pass_twiddles(int log2p) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, double2*> tables;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  double2*& slot = tables[{dev, log2p}];
  if (!slot) {
    const int p = 1 << log2p;
    std::vector<double2> h;
    h.reserve(twiddle_entries(p) + 1);
    const long double pi_l = 3.14159265358979323846264338327950288L;
    for (int ns = 1; ns < p; ns *= pass_radix(p, ns)) {
      const int r_ = pass_radix(p, ns);
      if (ns == 1) continue;
      for (int r = 1; r < r_; ++r)
        for (int k = 0; k < ns; ++k) {
          // w_{ns R}^{r k} = e^{-2 pi i r k / (ns R)}, phase reduced exactly
          const long long m = (long long)r * k % (long long)(ns * r_);
          const long double a = 2.0L * pi_l * (long double)m / (long double)(ns * r_);
          h.push_back(make_double2((double)cosl(a), (double)-sinl(a)));
        }
    }
    if (h.empty()) h.push_back(make_double2(1.0, 0.0));
    FLB_CUDA(cudaMalloc(&slot, h.size() * sizeof(double2)));
    FLB_CUDA(cudaMemcpy(slot, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  }
  return slot;
}

void fft_pow2(double2* data, double2* scratch, int log2p, size_t batch, bool inverse,
              cudaStream_t s) {
  if (log2p < 0 || log2p > kMaxLog2) fail(FL_RUNTIME_ERROR, "fft: length out of range");
  if (batch == 0) return;
  if (log2p <= kMaxSmemLog2) {
    fft_rows(data, log2p, batch, inverse, s);
    return;
  }
  const int lr = log2p / 2, lc = log2p - lr;
  const int R = 1 << lr, C = 1 << lc;
  const unsigned long long P = 1ull << log2p;
  // x[a1 + R a2] viewed as A[a2][a1] (C x R)
  for (size_t b0 = 0; b0 < batch; b0 += 65535) {
    const size_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    double2* d = data + b0 * P;
    double2* t = scratch + b0 * P;
    transpose(d, t, C, R, nb, 0, inverse, s);           // T1[a1][a2]
    fft_rows(t, lc, nb * R, inverse, s);                // Y[a1][b2]
    transpose(t, d, R, C, nb, P, inverse, s);           // T2[b2][a1] * w^{a1 b2}
    fft_rows(d, lr, nb * C, inverse, s);                // T2[b2][b1] = X[b2 + C b1]
    transpose(d, t, C, R, nb, 0, inverse, s);           // X[b1][b2]
    FLB_CUDA(cudaMemcpyAsync(d, t, nb * P * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace flb
