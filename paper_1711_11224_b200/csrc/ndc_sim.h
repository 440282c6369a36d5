// Simulation generators of the reference (simulation.hpp:36-191) with the image-sized
// work on the device.  See ndc_sim.cu for the bit-exactness argument.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ndc {

// Fails with NDC_ERR_NO_DEVICE / NDC_ERR_ARGUMENT unless `device` is a usable sm_100 GPU;
// makes it current.
void require_device(int device);

// Sequential std::mt19937_64 stream on the device: one CTA runs the 312-word twist in
// three parallel phases; the stream only moves forward, in whole twists of 312 words.
class Mt64Stream {
 public:
  static constexpr int kN = 312;
  Mt64Stream(uint64_t seed, cudaStream_t s);
  ~Mt64Stream();
  Mt64Stream(const Mt64Stream&) = delete;
  Mt64Stream& operator=(const Mt64Stream&) = delete;
  // Run `twists` twists; write their 312*twists tempered words to `out` (device) or,
  // for out == nullptr, discard them.
  void generate(size_t twists, uint64_t* out);
  size_t twists_done() const { return done_; }

 private:
  uint64_t* state_ = nullptr;  // device, 312 words
  cudaStream_t s_;
  size_t done_ = 0;
};

// Box-Muller over a device word buffer holding stream words [w0, w0 + nwords):
// dense[i] = (dense[i] + mean) + std_dev * z(s0 + i) for the samples s0 + i, i < n,
// whose word pair lies in the buffer (the reference's GaussianSource: sample 2p is
// r cos a, sample 2p+1 is r sin a, from words 2p and 2p+1).
cudaError_t launch_box_muller_add(double* dense, size_t n, size_t s0, const uint64_t* words, size_t w0,
                                  size_t nwords, double mean, double std_dev, cudaStream_t s);

// add_gaussian_noise (simulation.hpp:184-191) over one stream, applied to consecutive
// ranges of its samples: add(dense, n, s0) adds samples [s0, s0+n) to dense[0..n).
// Calls must come in increasing, non-overlapping s0 order; words before a range are
// generated and discarded, the buffer of the last chunk is kept for a pair that
// straddles two calls.
class GaussianNoise {
 public:
  GaussianNoise(uint64_t seed, double mean, double std_dev, cudaStream_t s);
  ~GaussianNoise();
  GaussianNoise(const GaussianNoise&) = delete;
  GaussianNoise& operator=(const GaussianNoise&) = delete;
  void add(double* dense, size_t n, size_t s0);

 private:
  static constexpr size_t kChunkTwists = 1 << 15;  // 10.2 M words (82 MB)
  Mt64Stream mt_;
  double mean_, std_;
  cudaStream_t s_;
  uint64_t* words_ = nullptr;
  size_t w0_ = 0, nw_ = 0;  // stream words held in words_
};

// Host-pointer entry points (ndc_capi.cu), each validated like the reference.
void sim_phantom_lines(int device, size_t rows, size_t cols, size_t n_lines, double intensity, double* out);
void sim_phantom_texture(int device, size_t rows, size_t cols, double* out);
void sim_gaussian_psf(int ndim, const size_t* ext, double sigma, double* out);
void sim_delta_psf(int ndim, const size_t* ext, double* out);
void sim_add_gaussian_noise(int device, size_t n, const double* in, double mean, double std_dev, uint64_t seed,
                            double* out);
void sim_mt19937_64(int device, uint64_t seed, size_t skip, size_t n, uint64_t* out);

}  // namespace ndc
