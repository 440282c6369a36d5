// Simulation generators (reference: simulation.hpp:36-191), image-sized work on the
// device, SURVEY §8f-4.
//
// Bit-exactness against the reference's host code:
//  * phantom_lines (36-70): the n_lines angles, sines, cosines and slopes are computed
//    on the host with the same libm calls (n_lines values); the per-pixel
//    `lround(cr + (c - cc) * slope)` runs on the device with explicitly rounded f64
//    operations (no FMA contraction), so every pixel equals the reference's.
//  * phantom_texture (72-94): the separable transcendentals sin(2*pi*2*r/rows) and
//    cos(2*pi*3*c/cols) are host tables (rows + cols values, same libm); the per-pixel
//    combination, disk test, fmod stripe and clamp are exact f64 device arithmetic.
//  * gaussian_psf / delta_psf (98-131): kernel-sized, host (same std::exp).
//  * add_gaussian_noise (154-191): the std::mt19937_64 word stream is generated on the
//    device bit for bit (integer arithmetic); Box-Muller uses the device's f64 log /
//    sin / cos, which agree with glibc's to a few ulp (tests pin <= 4 ulp), so noisy
//    samples agree to ~1e-15 relative.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ndc_plan.h"
#include "ndc_sim.h"

namespace ndc {

void require_device(int device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(NDC_ERR_NO_DEVICE, "ndconv_b200: no CUDA device (the device path has no CPU fallback)");
  }
  if (device < 0 || device >= ndev) fail(NDC_ERR_ARGUMENT, "ndconv_b200: bad device ordinal");
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  int major = 0;
  check_cuda(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device), "cudaDeviceGetAttribute");
  if (major != 10) fail(NDC_ERR_NO_DEVICE, "ndconv_b200: built for sm_100a");
}

namespace {

constexpr double kPi = 3.14159265358979323846;

// ---- mt19937_64 (the published MT19937-64 parameters, as std::mt19937_64) -------------
constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t mt_mix(uint64_t y) { return (y >> 1) ^ ((y & 1ull) ? kMatrixA : 0ull); }

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// One CTA of 320 threads; thread i < 312 owns state word i.  A twist is three phases:
//   A  i <  156: mt[i] = mt[i+156] ^ mix(hi(mt[i]) | lo(mt[i+1]))        (all old words)
//   B  156 <= i < 311: mt[i] = mt[i-156] ^ mix(hi(mt[i]) | lo(mt[i+1]))  (mt[i-156] new)
//      i == 311:       mt[311] = mt[155] ^ mix(hi(mt[311]) | lo(mt[0]))  (both new)
// which is the sequential recurrence's exact data flow.
__global__ void __launch_bounds__(320) mt_twist_kernel(uint64_t* __restrict__ state, size_t twists,
                                                       uint64_t* __restrict__ out) {
  __shared__ uint64_t mt[kMtN];
  const int i = threadIdx.x;
  if (i < kMtN) mt[i] = state[i];
  __syncthreads();
  for (size_t t = 0; t < twists; ++t) {
    uint64_t y = 0;
    if (i < kMtN - 1) y = (mt[i] & kUpper) | (mt[i + 1] & kLower);
    __syncthreads();
    if (i < kMtN - kMtM) mt[i] = mt[i + kMtM] ^ mt_mix(y);
    __syncthreads();
    if (i >= kMtN - kMtM && i < kMtN - 1) mt[i] = mt[i - (kMtN - kMtM)] ^ mt_mix(y);
    if (i == kMtN - 1) mt[i] = mt[kMtM - 1] ^ mt_mix((mt[i] & kUpper) | (mt[0] & kLower));
    __syncthreads();
    if (out != nullptr && i < kMtN) out[t * kMtN + i] = mt_temper(mt[i]);
  }
  if (i < kMtN) state[i] = mt[i];
}

// GaussianSource::next() (simulation.hpp:160-172) for the pair p = word pair (2p, 2p+1).
__global__ void box_muller_add_kernel(double* __restrict__ dense, size_t n, size_t s0,
                                      const uint64_t* __restrict__ words, size_t w0, size_t nwords, double mean,
                                      double std_dev) {
  const size_t p_lo = (s0 > w0 ? s0 : w0) / 2;  // first pair with a sample in range
  const size_t p_hi_s = (s0 + n + 1) / 2, p_hi_w = (w0 + nwords) / 2;
  const size_t p_hi = p_hi_s < p_hi_w ? p_hi_s : p_hi_w;
  for (size_t p = p_lo + blockIdx.x * size_t(blockDim.x) + threadIdx.x; p < p_hi;
       p += size_t(gridDim.x) * blockDim.x) {
    const uint64_t a1 = words[2 * p - w0], a2 = words[2 * p + 1 - w0];
    const double u1 = __dmul_rn(__dadd_rn(static_cast<double>(a1 >> 11), 1.0), 0x1.0p-53);
    const double u2 = __dmul_rn(static_cast<double>(a2 >> 11), 0x1.0p-53);
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    const double ang = __dmul_rn(2.0 * kPi, u2);
    double sn, cs;
    sincos(ang, &sn, &cs);
    const size_t se = 2 * p, so = 2 * p + 1;
    if (se >= s0 && se < s0 + n) {
      double& v = dense[se - s0];
      v = __dadd_rn(__dadd_rn(v, mean), __dmul_rn(std_dev, __dmul_rn(r, cs)));
    }
    if (so >= s0 && so < s0 + n) {
      double& v = dense[so - s0];
      v = __dadd_rn(__dadd_rn(v, mean), __dmul_rn(std_dev, __dmul_rn(r, sn)));
    }
  }
}

struct LineParam {
  int steep;      // 0: iterate columns (|dc| >= |dr|), 1: iterate rows
  double slope;
};

__global__ void phantom_lines_kernel(double* __restrict__ img, long rows, long cols, const LineParam* __restrict__ lp,
                                     double cr, double cc, double intensity) {
  const LineParam L = lp[blockIdx.y];
  const long len = L.steep ? rows : cols;
  for (long k = blockIdx.x * long(blockDim.x) + threadIdx.x; k < len; k += long(gridDim.x) * blockDim.x) {
    if (!L.steep) {
      const long r = lround(__dadd_rn(cr, __dmul_rn(__dadd_rn(static_cast<double>(k), -cc), L.slope)));
      if (r >= 0 && r < rows) img[r * cols + k] = intensity;
    } else {
      const long c = lround(__dadd_rn(cc, __dmul_rn(__dadd_rn(static_cast<double>(k), -cr), L.slope)));
      if (c >= 0 && c < cols) img[k * cols + c] = intensity;
    }
  }
}

__global__ void phantom_texture_kernel(double* __restrict__ img, long rows, long cols,
                                       const double* __restrict__ sin_r, const double* __restrict__ cos_c) {
  const double rn = static_cast<double>(rows), cn = static_cast<double>(cols);
  const double disk_r = __dmul_rn(0.15, fmin(rn, cn));
  const double disk_r2 = __dmul_rn(disk_r, disk_r);
  const double r_lo = __dmul_rn(0.65, rn), r_hi = __dmul_rn(0.78, rn);
  const double dr0 = __dmul_rn(0.3, rn), dc0 = __dmul_rn(0.35, cn);
  const long total = rows * cols;
  for (long f = blockIdx.x * long(blockDim.x) + threadIdx.x; f < total; f += long(gridDim.x) * blockDim.x) {
    const long r = f / cols, c = f - r * cols;
    const double rr = static_cast<double>(r), cc = static_cast<double>(c);
    double v = __dadd_rn(90.0, __dmul_rn(__dmul_rn(60.0, sin_r[r]), cos_c[c]));
    const double dr = __dadd_rn(rr, -dr0), dc = __dadd_rn(cc, -dc0);
    if (__dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dc, dc)) <= disk_r2) v = __dadd_rn(v, 90.0);
    if (rr >= r_lo && rr < r_hi && fmod(cc, 16.0) < 8.0) v = __dadd_rn(v, 70.0);
    img[f] = fmin(255.0, fmax(0.0, v));
  }
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { check_cuda(cudaMalloc(&p, n * sizeof(T) + 8), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

struct OwnedStream {
  cudaStream_t s = nullptr;
  OwnedStream() { check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate"); }
  ~OwnedStream() {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
};

int grid_for(size_t work, int block) {
  const size_t g = (work + block - 1) / block;
  return static_cast<int>(g < 148 * 16 ? (g == 0 ? 1 : g) : 148 * 16);
}

}  // namespace

// ---- mt19937_64 stream ---------------------------------------------------------------------
Mt64Stream::Mt64Stream(uint64_t seed, cudaStream_t s) : s_(s) {
  uint64_t init[kMtN];  // std::mersenne_twister_engine seeding (f = 6364136223846793005)
  init[0] = seed;
  for (int i = 1; i < kMtN; ++i) init[i] = 6364136223846793005ull * (init[i - 1] ^ (init[i - 1] >> 62)) + i;
  check_cuda(cudaMallocAsync(&state_, sizeof init, s_), "cudaMallocAsync");
  check_cuda(cudaMemcpyAsync(state_, init, sizeof init, cudaMemcpyHostToDevice, s_), "H2D");
  check_cuda(cudaStreamSynchronize(s_), "cudaStreamSynchronize");  // `init` is on this stack
}

Mt64Stream::~Mt64Stream() {
  if (state_) cudaFreeAsync(state_, s_);
}

void Mt64Stream::generate(size_t twists, uint64_t* out) {
  if (twists == 0) return;
  mt_twist_kernel<<<1, 320, 0, s_>>>(state_, twists, out);
  check_cuda(cudaGetLastError(), "mt_twist_kernel");
  done_ += twists;
}

cudaError_t launch_box_muller_add(double* dense, size_t n, size_t s0, const uint64_t* words, size_t w0,
                                  size_t nwords, double mean, double std_dev, cudaStream_t s) {
  if (n == 0 || nwords == 0) return cudaSuccess;
  box_muller_add_kernel<<<grid_for(nwords / 2, 256), 256, 0, s>>>(dense, n, s0, words, w0, nwords, mean, std_dev);
  return cudaGetLastError();
}

GaussianNoise::GaussianNoise(uint64_t seed, double mean, double std_dev, cudaStream_t s)
    : mt_(seed, s), mean_(mean), std_(std_dev), s_(s) {
  check_cuda(cudaMallocAsync(&words_, kChunkTwists * kMtN * 8, s_), "cudaMallocAsync");
}

GaussianNoise::~GaussianNoise() {
  if (words_) cudaFreeAsync(words_, s_);
}

void GaussianNoise::add(double* dense, size_t n, size_t s0) {
  if (n == 0) return;
  const size_t w_first = (s0 / 2) * 2, w_end = ((s0 + n + 1) / 2) * 2;
  // the pair straddling the previous call's end is still in the buffer
  check_cuda(launch_box_muller_add(dense, n, s0, words_, w0_, nw_, mean_, std_, s_), "box_muller");
  const size_t pos = mt_.twists_done() * kMtN;
  if (w_first > pos) mt_.generate((w_first - pos) / kMtN, nullptr);  // skip whole twists
  while (mt_.twists_done() * kMtN < w_end) {
    const size_t w0 = mt_.twists_done() * kMtN;
    const size_t left = (w_end - w0 + kMtN - 1) / kMtN;
    const size_t t = left < kChunkTwists ? left : kChunkTwists;
    mt_.generate(t, words_);
    w0_ = w0;
    nw_ = t * kMtN;
    check_cuda(launch_box_muller_add(dense, n, s0, words_, w0_, nw_, mean_, std_, s_), "box_muller");
  }
}

// ---- host-pointer entry points -----------------------------------------------------------
void sim_phantom_lines(int device, size_t rows, size_t cols, size_t n_lines, double intensity, double* out) {
  if (rows < 3 || cols < 3) fail(NDC_ERR_SHAPE, "phantom_lines: size must be at least 3x3");
  if (n_lines < 1) fail(NDC_ERR_CONFIG, "phantom_lines: need at least one line");
  require_device(device);
  const double cr = static_cast<double>(rows / 2), cc = static_cast<double>(cols / 2);
  std::vector<LineParam> lp(n_lines);
  for (size_t i = 0; i < n_lines; ++i) {  // simulation.hpp:47-50, host libm
    const double theta = kPi * static_cast<double>(i) / static_cast<double>(n_lines);
    const double dr = std::sin(theta), dc = std::cos(theta);
    lp[i] = std::abs(dc) >= std::abs(dr) ? LineParam{0, dr / dc} : LineParam{1, dc / dr};
  }
  OwnedStream st;
  DevBuf<double> img(rows * cols);
  DevBuf<LineParam> dlp(n_lines);
  check_cuda(cudaMemsetAsync(img.p, 0, rows * cols * 8, st.s), "cudaMemset");
  check_cuda(cudaMemcpyAsync(dlp.p, lp.data(), n_lines * sizeof(LineParam), cudaMemcpyHostToDevice, st.s), "H2D");
  const size_t len = rows > cols ? rows : cols;
  if (n_lines > 65535) fail(NDC_ERR_UNSUPPORTED, "phantom_lines: at most 65535 lines");
  dim3 grid(static_cast<unsigned>((len + 255) / 256), static_cast<unsigned>(n_lines));
  phantom_lines_kernel<<<grid, 256, 0, st.s>>>(img.p, static_cast<long>(rows), static_cast<long>(cols), dlp.p, cr,
                                               cc, intensity);
  check_cuda(cudaGetLastError(), "phantom_lines_kernel");
  check_cuda(cudaMemcpyAsync(out, img.p, rows * cols * 8, cudaMemcpyDeviceToHost, st.s), "D2H");
  check_cuda(cudaStreamSynchronize(st.s), "cudaStreamSynchronize");
}

void sim_phantom_texture(int device, size_t rows, size_t cols, double* out) {
  if (rows < 3 || cols < 3) fail(NDC_ERR_SHAPE, "phantom_texture: size must be at least 3x3");
  require_device(device);
  const double rn = static_cast<double>(rows), cn = static_cast<double>(cols);
  std::vector<double> sr(rows), cc(cols);  // simulation.hpp:84-85, host libm
  for (size_t r = 0; r < rows; ++r) sr[r] = std::sin(2 * kPi * 2.0 * static_cast<double>(r) / rn);
  for (size_t c = 0; c < cols; ++c) cc[c] = std::cos(2 * kPi * 3.0 * static_cast<double>(c) / cn);
  OwnedStream st;
  DevBuf<double> img(rows * cols), dsr(rows), dcc(cols);
  check_cuda(cudaMemcpyAsync(dsr.p, sr.data(), rows * 8, cudaMemcpyHostToDevice, st.s), "H2D");
  check_cuda(cudaMemcpyAsync(dcc.p, cc.data(), cols * 8, cudaMemcpyHostToDevice, st.s), "H2D");
  phantom_texture_kernel<<<grid_for(rows * cols, 256), 256, 0, st.s>>>(img.p, static_cast<long>(rows),
                                                                       static_cast<long>(cols), dsr.p, dcc.p);
  check_cuda(cudaGetLastError(), "phantom_texture_kernel");
  check_cuda(cudaMemcpyAsync(out, img.p, rows * cols * 8, cudaMemcpyDeviceToHost, st.s), "D2H");
  check_cuda(cudaStreamSynchronize(st.s), "cudaStreamSynchronize");
}

namespace {
size_t checked_kernel_count(int ndim, const size_t* ext, const char* what) {
  if (ndim < 1) fail(NDC_ERR_SHAPE, "Shape: need at least one dimension");
  size_t n = 1;
  for (int i = 0; i < ndim; ++i) {
    if (ext[i] == 0) fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
    if (ext[i] % 2 == 0) fail(NDC_ERR_SHAPE, std::string(what) + ": extents must be odd");
    n *= ext[i];
  }
  return n;
}
}  // namespace

void sim_gaussian_psf(int ndim, const size_t* ext, double sigma, double* out) {
  if (!(sigma > 0)) fail(NDC_ERR_NUMERIC, "gaussian_psf: sigma must be positive");
  const size_t n = checked_kernel_count(ndim, ext, "gaussian_psf");
  std::vector<size_t> idx(ndim, 0);
  double total = 0.0;
  for (size_t f = 0; f < n; ++f) {  // simulation.hpp:108-118, storage order
    double d2 = 0.0;
    for (int i = 0; i < ndim; ++i) {
      const double d = static_cast<double>(idx[i]) - static_cast<double>((ext[i] - 1) / 2);
      d2 += d * d;
    }
    out[f] = std::exp(-d2 / (2.0 * sigma * sigma));
    total += out[f];
    for (int i = ndim - 1; i >= 0; --i) {
      if (++idx[i] < ext[i]) break;
      idx[i] = 0;
    }
  }
  for (size_t f = 0; f < n; ++f) out[f] /= total;
}

void sim_delta_psf(int ndim, const size_t* ext, double* out) {
  const size_t n = checked_kernel_count(ndim, ext, "Kernel");
  std::memset(out, 0, n * 8);
  size_t f = 0;
  for (int i = 0; i < ndim; ++i) f = f * ext[i] + ext[i] / 2;
  out[f] = 1.0;
}

void sim_add_gaussian_noise(int device, size_t n, const double* in, double mean, double std_dev, uint64_t seed,
                            double* out) {
  if (std_dev < 0) fail(NDC_ERR_NUMERIC, "add_gaussian_noise: std_dev must be >= 0");
  require_device(device);
  if (n == 0) return;
  OwnedStream st;
  DevBuf<double> d(n);
  check_cuda(cudaMemcpyAsync(d.p, in, n * 8, cudaMemcpyHostToDevice, st.s), "H2D");
  {
    GaussianNoise noise(seed, mean, std_dev, st.s);
    noise.add(d.p, n, 0);
  }
  check_cuda(cudaMemcpyAsync(out, d.p, n * 8, cudaMemcpyDeviceToHost, st.s), "D2H");
  check_cuda(cudaStreamSynchronize(st.s), "cudaStreamSynchronize");
}

void sim_mt19937_64(int device, uint64_t seed, size_t skip, size_t n, uint64_t* out) {
  require_device(device);
  if (n == 0) return;
  OwnedStream st;
  Mt64Stream mt(seed, st.s);
  mt.generate(skip / kMtN, nullptr);
  const size_t first = mt.twists_done() * kMtN;
  const size_t twists = (skip + n - first + kMtN - 1) / kMtN;
  DevBuf<uint64_t> w(twists * kMtN);
  mt.generate(twists, w.p);
  check_cuda(cudaMemcpyAsync(out, w.p + (skip - first), n * 8, cudaMemcpyDeviceToHost, st.s), "D2H");
  check_cuda(cudaStreamSynchronize(st.s), "cudaStreamSynchronize");
}

}  // namespace ndc
