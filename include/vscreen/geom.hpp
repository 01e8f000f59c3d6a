// vscreen/geom.hpp — the drop-in's FP64 vector and quaternion value types.
//
// Source-compatible with the reference's geometry header
// (proj/include/vscreen/geom.hpp:7-54): the same member names, operators and
// rotation formula, because callers construct these types directly and the
// dock contract (pose convention x = R(q) y + t) is defined on them.
#pragma once

#include <cmath>

namespace vscreen {

struct Vec3 {
  double x = 0.0;
  double y = 0.0;
  double z = 0.0;

  Vec3& operator+=(const Vec3& v) {
    x += v.x, y += v.y, z += v.z;
    return *this;
  }
  Vec3& operator-=(const Vec3& v) {
    x -= v.x, y -= v.y, z -= v.z;
    return *this;
  }
  Vec3 operator+(const Vec3& v) const { return Vec3{x + v.x, y + v.y, z + v.z}; }
  Vec3 operator-(const Vec3& v) const { return Vec3{x - v.x, y - v.y, z - v.z}; }
  Vec3 operator*(double k) const { return Vec3{x * k, y * k, z * k}; }
  Vec3 operator/(double k) const { return Vec3{x / k, y / k, z / k}; }

  [[nodiscard]] double dot(const Vec3& v) const { return x * v.x + y * v.y + z * v.z; }
  [[nodiscard]] Vec3 cross(const Vec3& v) const;
  [[nodiscard]] double norm2() const { return dot(*this); }
  [[nodiscard]] double norm() const { return std::sqrt(norm2()); }
  // zero stays zero
  [[nodiscard]] Vec3 normalized() const;
};

inline Vec3 Vec3::cross(const Vec3& v) const {
  return Vec3{y * v.z - z * v.y, z * v.x - x * v.z, x * v.y - y * v.x};
}

inline Vec3 Vec3::normalized() const {
  const double len = norm();
  if (!(len > 0.0)) return Vec3{};
  return *this / len;
}

inline Vec3 operator*(double k, const Vec3& v) { return v * k; }

inline double distance(const Vec3& a, const Vec3& b) { return (a - b).norm(); }

// (w, x, y, z); rotate() assumes a unit quaternion
struct Quat {
  double w = 1.0;
  double x = 0.0;
  double y = 0.0;
  double z = 0.0;

  [[nodiscard]] double norm() const { return std::sqrt(w * w + x * x + y * y + z * z); }
  [[nodiscard]] Quat normalized() const;
  // v' = v + 2w (u x v) + 2 u x (u x v) with u = (x, y, z)
  [[nodiscard]] Vec3 rotate(const Vec3& v) const;
  static Quat from_axis_angle(const Vec3& unit_axis, double angle);
};

inline Quat Quat::normalized() const {
  const double len = norm();
  return Quat{w / len, x / len, y / len, z / len};
}

inline Vec3 Quat::rotate(const Vec3& v) const {
  const Vec3 u{x, y, z};
  const Vec3 t = u.cross(v);
  return v + 2.0 * w * t + 2.0 * u.cross(t);
}

inline Quat Quat::from_axis_angle(const Vec3& unit_axis, double angle) {
  const double half = 0.5 * angle;
  const double s = std::sin(half);
  return Quat{std::cos(half), unit_axis.x * s, unit_axis.y * s, unit_axis.z * s};
}

}  // namespace vscreen
