// wfn1.h — WFN1 orbital files (reference model.hpp:236-339), host side.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace lrgw_host {

// Any WFN1 failure; the message is the reference's io_error text.
struct Wfn1Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Wfn1Header {
  int dims[3] = {0, 0, 0};
  double cell[3] = {0, 0, 0};
  long long n_r = 0;
  int n_v = 0, n_c = 0;
  long long payload_offset = 0;  // byte offset of psi
};

// The header the reference's save_system writes (nlohmann::json::dump bytes).
std::string wfn1_header_json(const int dims[3], const double cell[3], int n_v, int n_c);
// Parse and validate the header with load_system's checks and messages.
Wfn1Header wfn1_read_header(const char* path);
// n doubles at byte offset `offset` (throws "truncated payload reading <what>").
void wfn1_read_payload(const char* path, long long offset, double* dst, size_t n, const char* what);
void wfn1_write(const char* path, const int dims[3], const double cell[3], int n_v, int n_c, const double* psi,
                const double* energies, const double* vxc);

}  // namespace lrgw_host
