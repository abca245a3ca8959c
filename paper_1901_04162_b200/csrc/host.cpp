// host.cpp -- host-side setup code of libgk: quadrature rules and the
// benchmark's mesh generators.  Compiled with -ffp-contract=off so the rules
// and meshes are bit-identical to the reference's (quadrature.hpp,
// mesh.hpp); this is input setup, excluded from fill timing like the
// reference's (matfill.hpp:139-141).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "gk_internal.h"

namespace gk {

// symmetric triangle rules, quadrature.hpp:35-76
void triangle_rule(int m, double* b0, double* b1, double* b2, double* w) {
  struct P { double b0, b1, b2, w; };
  static const P r1[] = {{1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, 1.0}};
  static const P r3[] = {{2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0, 1.0 / 3.0},
                         {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0, 1.0 / 3.0},
                         {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0, 1.0 / 3.0}};
  static const P r4[] = {{1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, -27.0 / 48.0},
                         {0.6, 0.2, 0.2, 25.0 / 48.0},
                         {0.2, 0.6, 0.2, 25.0 / 48.0},
                         {0.2, 0.2, 0.6, 25.0 / 48.0}};
  // degree-5 / degree-4 symmetric rules (Dunavant), 15 significant digits
  constexpr double a6 = 0.108103018168070, b6 = 0.445948490915965, w6a = 0.223381589678011;
  constexpr double c6 = 0.816847572980459, d6 = 0.091576213509771, w6b = 0.109951743655322;
  static const P r6[] = {{a6, b6, b6, w6a}, {b6, a6, b6, w6a}, {b6, b6, a6, w6a},
                         {c6, d6, d6, w6b}, {d6, c6, d6, w6b}, {d6, d6, c6, w6b}};
  constexpr double a7 = 0.059715871789770, b7 = 0.470142064105115, w7a = 0.132394152788506;
  constexpr double c7 = 0.797426985353087, d7 = 0.101286507323456, w7b = 0.125939180544827;
  static const P r7[] = {{1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, 0.225},
                         {a7, b7, b7, w7a}, {b7, a7, b7, w7a}, {b7, b7, a7, w7a},
                         {c7, d7, d7, w7b}, {d7, c7, d7, w7b}, {d7, d7, c7, w7b}};
  const P* r = nullptr;
  switch (m) {
    case 1: r = r1; break;
    case 3: r = r3; break;
    case 4: r = r4; break;
    case 6: r = r6; break;
    case 7: r = r7; break;
    default: fail(GK_ERR_INVALID_ARGUMENT, "triangle_rule: unsupported point count (use 1, 3, 4, 6, 7)");
  }
  for (int i = 0; i < m; ++i) {
    b0[i] = r[i].b0;
    b1[i] = r[i].b1;
    b2[i] = r[i].b2;
    w[i] = r[i].w;
  }
}

// Gauss-Legendre on [0,1] by Newton on the Legendre recurrence,
// quadrature.hpp:85-110 (same iteration, same stopping rule)
void gauss_legendre_unit(int n, double* xs, double* ws) {
  if (n < 1) fail(GK_ERR_INVALID_ARGUMENT, "gauss_legendre_unit: n must be >= 1");
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double x = std::cos(kPi * (static_cast<double>(i) + 0.75) / (static_cast<double>(n) + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int j = 2; j <= n; ++j) {
        const double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / static_cast<double>(j);
        p0 = p1;
        p1 = p2;
      }
      dp = n == 1 ? 1.0 : static_cast<double>(n) * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    xs[i] = (1.0 - x) / 2.0;
    ws[i] = w / 2.0;
    xs[n - 1 - i] = (1.0 + x) / 2.0;
    ws[n - 1 - i] = w / 2.0;
  }
}

namespace {

struct V3 {
  double x, y, z;
};
V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 scale(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
double norm(V3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

}  // namespace

// icosphere, mesh.hpp:154-202: midpoints created on first sight, children in
// the order {t0,ab,ca},{t1,bc,ab},{t2,ca,bc},{ab,bc,ca}, projection last
void sphere_mesh(double radius, int subdivisions, std::vector<double>& verts,
                 std::vector<uint32_t>& tris) {
  if (!(radius > 0.0)) fail(GK_ERR_INVALID_ARGUMENT, "generate_sphere_mesh: radius must be > 0");
  if (subdivisions < 0 || subdivisions > 6)
    fail(GK_ERR_INVALID_ARGUMENT, "generate_sphere_mesh: subdivisions must be in [0, 6]");
  const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<V3> v = {{-1, phi, 0}, {1, phi, 0},   {-1, -phi, 0}, {1, -phi, 0},
                       {0, -1, phi}, {0, 1, phi},   {0, -1, -phi}, {0, 1, -phi},
                       {phi, 0, -1}, {phi, 0, 1},   {-phi, 0, -1}, {-phi, 0, 1}};
  std::vector<uint32_t> t = {0, 11, 5, 0, 5,  1,  0,  1, 7,  0, 7, 10, 0, 10, 11,
                             1, 5,  9, 5, 11, 4,  11, 10, 2, 10, 7, 6,  7, 1,  8,
                             3, 9,  4, 3, 4,  2,  3,  2, 6,  3, 6, 8,  3, 8,  9,
                             4, 9,  5, 2, 4,  11, 6,  2, 10, 8, 6, 7,  9, 8,  1};
  for (int level = 0; level < subdivisions; ++level) {
    std::unordered_map<uint64_t, uint32_t> mid;
    mid.reserve(t.size());
    auto midpoint = [&](uint32_t a, uint32_t b) {
      const uint64_t key = a < b ? (uint64_t(a) << 32 | b) : (uint64_t(b) << 32 | a);
      const auto it = mid.find(key);
      if (it != mid.end()) return it->second;
      v.push_back(scale(add(v[a], v[b]), 0.5));
      const auto idx = static_cast<uint32_t>(v.size() - 1);
      mid.emplace(key, idx);
      return idx;
    };
    std::vector<uint32_t> next;
    next.reserve(t.size() * 4);
    for (size_t i = 0; i < t.size(); i += 3) {
      const uint32_t a = t[i], b = t[i + 1], c = t[i + 2];
      const uint32_t ab = midpoint(a, b), bc = midpoint(b, c), ca = midpoint(c, a);
      const uint32_t kids[12] = {a, ab, ca, b, bc, ab, c, ca, bc, ab, bc, ca};
      next.insert(next.end(), kids, kids + 12);
    }
    t.swap(next);
  }
  verts.resize(3 * v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    const V3 p = scale(v[i], radius / norm(v[i]));
    verts[3 * i] = p.x;
    verts[3 * i + 1] = p.y;
    verts[3 * i + 2] = p.z;
  }
  tris.swap(t);
}

void plate_mesh(double side, int cells, std::vector<double>& verts, std::vector<uint32_t>& tris) {
  if (!(side > 0.0) || cells < 1) fail(GK_ERR_INVALID_ARGUMENT, "plate_mesh: need side > 0, cells >= 1");
  const size_t c1 = static_cast<size_t>(cells) + 1;
  verts.assign(3 * c1 * c1, 0.0);
  for (size_t j = 0; j < c1; ++j)
    for (size_t i = 0; i < c1; ++i) {
      verts[3 * (j * c1 + i)] = side * static_cast<double>(i) / static_cast<double>(cells);
      verts[3 * (j * c1 + i) + 1] = side * static_cast<double>(j) / static_cast<double>(cells);
    }
  tris.clear();
  tris.reserve(6 * static_cast<size_t>(cells) * cells);
  for (size_t j = 0; j < static_cast<size_t>(cells); ++j)
    for (size_t i = 0; i < static_cast<size_t>(cells); ++i) {
      const auto v00 = static_cast<uint32_t>(j * c1 + i), v10 = v00 + 1;
      const auto v01 = static_cast<uint32_t>(v00 + c1), v11 = v01 + 1;
      const uint32_t two[6] = {v00, v10, v11, v00, v11, v01};
      tris.insert(tris.end(), two, two + 6);
    }
}

void jitter(double* v, size_t nv, uint64_t seed, double amp) {
  uint64_t s = seed;
  for (size_t i = 0; i < 3 * nv; ++i) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
    v[i] += amp * (2.0 * u - 1.0);
  }
}

// TriangleMesh::validate (mesh.hpp:46-57)
void validate_mesh(const double* v, size_t nv, const uint32_t* t, size_t nt) {
  for (size_t i = 0; i < nt; ++i) {
    for (int c = 0; c < 3; ++c)
      if (t[3 * i + c] >= nv)
        fail(GK_ERR_INVALID_ARGUMENT, "TriangleMesh: triangle " + std::to_string(i) +
                                          " references vertex " + std::to_string(t[3 * i + c]) +
                                          " out of range");
    const double* a = v + 3 * static_cast<size_t>(t[3 * i]);
    const double* b = v + 3 * static_cast<size_t>(t[3 * i + 1]);
    const double* c = v + 3 * static_cast<size_t>(t[3 * i + 2]);
    const double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
    const double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
    const double cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
    const double area = 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
    if (!(area > 1e-12))
      fail(GK_ERR_INVALID_ARGUMENT,
           "TriangleMesh: triangle " + std::to_string(i) + " is degenerate (area <= 1e-12)");
  }
}

}  // namespace gk
