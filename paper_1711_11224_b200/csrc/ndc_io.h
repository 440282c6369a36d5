// Host-side tensor file formats (ndc_io.cu).
#pragma once

#include <cstddef>
#include <string>
#include <vector>

namespace ndc {

struct NdtHeader {
  std::vector<size_t> ext;
  size_t count = 0;
  size_t payload_offset = 0;  // bytes from file start to the first f64
};

// Parses and validates the header line and the payload size (truncated / trailing
// data -> NDC_ERR_FORMAT), without reading the payload.
NdtHeader read_ndtensor_header(const std::string& path);
void read_ndtensor(const std::string& path, double* out, size_t capacity, NdtHeader* hdr);
void check_finite_payload(const double* v, size_t n, size_t first_index);
std::string ndtensor_header_line(const std::vector<size_t>& ext);
void write_ndtensor(const std::string& path, const std::vector<size_t>& ext, const double* data);
void read_pgm(const std::string& path, std::vector<double>* data, size_t* height, size_t* width);
void write_pgm(const std::string& path, size_t height, size_t width, const double* data, bool clamp);

}  // namespace ndc
