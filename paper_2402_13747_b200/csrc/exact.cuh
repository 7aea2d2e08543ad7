// exact.cuh — FP64 3-vector arithmetic in the reference's evaluation order.
//
// The reference computes with Eigen::Vector3d (proj/include/pcray/geometry.hpp:13).
// Bit-exact parity needs the same operation sequence:
//   dot(a,b)     = (a0*b0 + a1*b1) + a2*b2       squaredNorm = dot(a,a)
//   norm         = sqrt(squaredNorm)
//   normalized   = z = squaredNorm; z > 0 ? v / sqrt(z) : v   (true division)
//   cross        = (a1*b2 - a2*b1, a2*b0 - a0*b2, a0*b1 - a1*b0)
//   std::min/max/clamp as the libstdc++ ternaries (argument order matters for ±0)
// Every translation unit that includes this is compiled with --fmad=false
// (device) and -ffp-contract=off (host) so no a*b+c is fused.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define PCR_HD __host__ __device__ __forceinline__
#else
#define PCR_HD inline
#endif

namespace pcr {

struct V3 {
  double x, y, z;
};

PCR_HD V3 v3(double x, double y, double z) { return V3{x, y, z}; }
PCR_HD V3 load3(const double* p) { return V3{p[0], p[1], p[2]}; }
PCR_HD void store3(double* p, const V3& v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
PCR_HD double comp(const V3& v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }
PCR_HD void set_comp(V3& v, int a, double s) {
  if (a == 0) v.x = s;
  else if (a == 1) v.y = s;
  else v.z = s;
}

PCR_HD V3 operator+(const V3& a, const V3& b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
PCR_HD V3 operator-(const V3& a, const V3& b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
PCR_HD V3 operator-(const V3& a) { return V3{-a.x, -a.y, -a.z}; }
// scalar * vector (Eigen: per-coefficient s * v_i)
PCR_HD V3 operator*(double s, const V3& v) { return V3{s * v.x, s * v.y, s * v.z}; }
PCR_HD V3 operator*(const V3& v, double s) { return V3{v.x * s, v.y * s, v.z * s}; }
PCR_HD V3 operator/(const V3& v, double s) { return V3{v.x / s, v.y / s, v.z / s}; }
PCR_HD bool operator==(const V3& a, const V3& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
PCR_HD bool operator!=(const V3& a, const V3& b) { return !(a == b); }

PCR_HD double dot(const V3& a, const V3& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
PCR_HD double sqnorm(const V3& a) { return dot(a, a); }
PCR_HD double norm(const V3& a) { return sqrt(sqnorm(a)); }
// norm(v) <= y for y > 0, decided on the squared norm when it is clear of the rounding
// band: a <= y²(1-1e-12) implies sqrt_rn(a) < y and a >= y²(1+1e-12) implies
// sqrt_rn(a) > y (each rounding is within 2^-53 relative); the sqrt runs only inside
// the band, so the result equals the reference's `v.norm() <= y` bit for bit.
PCR_HD bool norm_le(const V3& v, double y) {
  const double a = sqnorm(v);
  const double yy = y * y;
  if (a <= yy * (1.0 - 1e-12)) return true;
  if (a >= yy * (1.0 + 1e-12)) return false;
  return sqrt(a) <= y;
}
PCR_HD V3 normalized(const V3& v) {
  const double z = sqnorm(v);
  return z > 0.0 ? v / sqrt(z) : v;
}
PCR_HD V3 cross(const V3& a, const V3& b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// Eigen isZero() with dummy_precision 1e-12 for double
PCR_HD bool is_zero(const V3& v) {
  return fabs(v.x) <= 1e-12 && fabs(v.y) <= 1e-12 && fabs(v.z) <= 1e-12;
}

// libstdc++ std::min / std::max / std::clamp
template <typename T>
PCR_HD T smin(T a, T b) { return (b < a) ? b : a; }
template <typename T>
PCR_HD T smax(T a, T b) { return (a < b) ? b : a; }
template <typename T>
PCR_HD T sclamp(T v, T lo, T hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

// tracer.cpp:94-97 safe_normalized: divide by the norm (not normalized()).
constexpr double kTiny = 1e-12;
PCR_HD V3 safe_normalized(const V3& v) {
  const double n = norm(v);
  return n > kTiny ? v / n : V3{0.0, 0.0, 0.0};
}

// geometry.hpp:33-37 angle_between = atan2(|a x b|, a.b)
PCR_HD double angle_between(const V3& a, const V3& b) {
  const double c = dot(a, b);
  const double s = norm(cross(a, b));
  return atan2(s, c);
}

// surface.cpp:164-177 local_frame: least-aligned axis, ties toward the higher index.
PCR_HD void local_frame(const V3& n, V3& u, V3& v) {
  int axis = 0;
  double best = fabs(n.x);
  if (fabs(n.y) <= best) {
    best = fabs(n.y);
    axis = 1;
  }
  if (fabs(n.z) <= best) {
    best = fabs(n.z);
    axis = 2;
  }
  const V3 a = axis == 0 ? V3{1, 0, 0} : (axis == 1 ? V3{0, 1, 0} : V3{0, 0, 1});
  u = normalized(cross(a, n));
  v = cross(n, u);
}

}  // namespace pcr
