// pcb200_quantize.hpp — the reference's quantizer API (/root/reference/proj/include/pcadmm/
// quantize.hpp:13-71) over the C ABI: gamma2 / gamma1 (scalar and vector), the combined integer
// update and its inverse run on the B200 (pcb_quantize, pcb_combined_update,
// pcb_inverse_quantize_x: FP64 in the reference's operation order, no contraction).  degamma* and
// widen_bounds are the reference's scalar host formulas (session set-up, no per-element batch).
#pragma once

#include <vector>

#include "pcb200_pcadmm.hpp"

namespace pcadmm {

struct QuantSpec {
  double z_min = 0.0;
  double z_max = 0.0;
  double delta = 1e15;
  double range() const { return z_max - z_min; }
};

struct ClampStats {
  u64 low = 0, high = 0;
  u64 total() const { return low + high; }
};

u64 gamma2(double v, const QuantSpec& s, ClampStats* clamps = nullptr);
u128 gamma1(double v, const QuantSpec& s, ClampStats* clamps = nullptr);
double degamma2(u64 q, const QuantSpec& s);
double degamma1(u128 q, const QuantSpec& s);
std::vector<u64> gamma2_vec(const std::vector<double>& v, const QuantSpec& s, ClampStats* clamps = nullptr);
std::vector<u128> gamma1_vec(const std::vector<double>& v, const QuantSpec& s, ClampStats* clamps = nullptr);
std::vector<u128> combined_quantized_update(const std::vector<u128>& q_alpha, const std::vector<std::vector<u64>>& q_b,
                                            const std::vector<u64>& q_z, const std::vector<u64>& q_negv);
std::vector<double> inverse_quantize_x(const std::vector<u128>& q, const std::vector<u64>& q_b_rowsum,
                                       const std::vector<u64>& q_z, const std::vector<u64>& q_negv,
                                       const QuantSpec& s);
QuantSpec widen_bounds(double lo, double hi, double margin, double delta);

}  // namespace pcadmm
