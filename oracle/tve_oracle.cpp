// tve_oracle.cpp — bodies of the CPU fp64 oracle.  TEST INFRASTRUCTURE ONLY
// (see tve_oracle.hpp).  Every function cites the reference declaration it
// restates and the SPEC.md formula it implements.
#include "tve_oracle.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <sstream>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace tve_oracle {

// ============================================================ linear algebra
Mat3 operator*(const Mat3& a, const Mat3& b) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += a.m[i][k] * b.m[k][j];
            r.m[i][j] = s;
        }
    return r;
}
Mat3 operator+(const Mat3& a, const Mat3& b) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] + b.m[i][j];
    return r;
}
Mat3 operator-(const Mat3& a, const Mat3& b) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] - b.m[i][j];
    return r;
}
Mat3 operator*(double s, const Mat3& a) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = s * a.m[i][j];
    return r;
}
Vec3 operator*(const Mat3& a, const Vec3& x) {
    Vec3 r;
    for (int i = 0; i < 3; ++i) r[i] = a.m[i][0] * x[0] + a.m[i][1] * x[1] + a.m[i][2] * x[2];
    return r;
}
Mat3 transpose(const Mat3& a) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}
double det(const Mat3& a) {
    return a.m[0][0] * (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) -
           a.m[0][1] * (a.m[1][0] * a.m[2][2] - a.m[1][2] * a.m[2][0]) +
           a.m[0][2] * (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]);
}
// Gauss-Jordan with partial pivoting: deliberately a different algorithm from
// the adjugate form the CUDA kernels use, so the two cross-check each other.
static Mat3 inverse_core(const Mat3& a, bool* bad) {
    double w[3][6];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            w[i][j] = a.m[i][j];
            w[i][3 + j] = (i == j) ? 1.0 : 0.0;
        }
    for (int c = 0; c < 3; ++c) {
        int p = c;
        for (int r = c + 1; r < 3; ++r)
            if (std::fabs(w[r][c]) > std::fabs(w[p][c])) p = r;
        if (w[p][c] == 0.0) {
            *bad = true;
            Mat3 r;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) r.m[i][j] = std::numeric_limits<double>::quiet_NaN();
            return r;
        }
        if (p != c)
            for (int j = 0; j < 6; ++j) std::swap(w[p][j], w[c][j]);
        const double inv = 1.0 / w[c][c];
        for (int j = 0; j < 6; ++j) w[c][j] *= inv;
        for (int r = 0; r < 3; ++r) {
            if (r == c) continue;
            const double f = w[r][c];
            if (f != 0.0)
                for (int j = 0; j < 6; ++j) w[r][j] -= f * w[c][j];
        }
    }
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = w[i][3 + j];
    return r;
}
Mat3 inverse(const Mat3& a) {
    bool bad = false;
    Mat3 r = inverse_core(a, &bad);
    if (bad) throw ValidationError("singular 3x3 matrix");
    return r;
}
double trace(const Mat3& a) { return a.m[0][0] + a.m[1][1] + a.m[2][2]; }
Mat3 outer(const Vec3& a, const Vec3& b) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a[i] * b[j];
    return r;
}

static double sym_max_eigenvalue(const Mat3& A) {
    // Cyclic Jacobi on a symmetric 3x3.
    double a[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) a[i][j] = 0.5 * (A.m[i][j] + A.m[j][i]);
    for (int sweep = 0; sweep < 50; ++sweep) {
        double off = std::fabs(a[0][1]) + std::fabs(a[0][2]) + std::fabs(a[1][2]);
        if (off < 1e-300) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                if (a[p][q] == 0) continue;
                double theta = (a[q][q] - a[p][p]) / (2 * a[p][q]);
                double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
                double c = 1 / std::sqrt(t * t + 1), s = t * c;
                for (int k = 0; k < 3; ++k) {
                    double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
            }
    }
    return std::max(a[0][0], std::max(a[1][1], a[2][2]));
}

// ============================================================ mesh (mesh.hpp:39-100)
// Corner signs of the standard brick ordering: bottom face CCW, top face CCW.
static const int kH8Sign[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                                  {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
// Reference gradients of the linear tet shape functions N1 = 1-xi-eta-zeta, N2..N4 = xi, eta, zeta.
static const int kT4Xi[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
// Hourglass base vectors h1 = eta*zeta, h2 = zeta*xi, h3 = xi*eta, h4 = xi*eta*zeta.
static const int kHg[4][8] = {{1, 1, -1, -1, -1, -1, 1, 1},
                              {1, -1, -1, 1, -1, 1, 1, -1},
                              {1, -1, 1, -1, 1, -1, 1, -1},
                              {-1, 1, -1, 1, 1, -1, 1, -1}};

// mesh.hpp:80-84 hourglass_basis_for_element: gamma_hat = h - (X h)^T G, then unit 2-norm.
void hourglass_basis_for_element(const double* coords, const double* grad, double* gamma) {
    for (int al = 0; al < 4; ++al) {
        double c[3] = {0, 0, 0};
        for (int a = 0; a < 8; ++a)
            for (int i = 0; i < 3; ++i) c[i] += coords[a * 3 + i] * kHg[al][a];
        double g[8], nrm = 0;
        for (int a = 0; a < 8; ++a) {
            double cg = c[0] * grad[a * 3 + 0] + c[1] * grad[a * 3 + 1] + c[2] * grad[a * 3 + 2];
            g[a] = kHg[al][a] - cg;
            nrm += g[a] * g[a];
        }
        nrm = std::sqrt(nrm);
        for (int a = 0; a < 8; ++a) gamma[al * 8 + a] = g[a] / nrm;
    }
}

// mesh.hpp:81-83 precompute.
PrecomputedMesh precompute(const Mesh& mesh, double density, double ref_specific_heat) {
    PrecomputedMesh pre;
    pre.kind = mesh.kind;
    const int N = mesh.node_count(), E = mesh.element_count(), nn = mesh.nodes_per_elem();
    pre.num_nodes = N;
    pre.num_elements = E;
    pre.shape_gradients.assign((size_t)E * 3 * nn, 0.0);
    pre.ref_volume.assign(E, 0.0);
    if (mesh.kind == ElementKind::H8) {
        pre.det_jacobian.assign(E, 0.0);
        pre.hourglass_basis.assign((size_t)E * 32, 0.0);
    }
    for (int e = 0; e < E; ++e) {
        const auto& el = mesh.elements[e];
        for (int a = 0; a < nn; ++a)
            if (el[a] < 0 || el[a] >= N)
                throw ValidationError("element " + std::to_string(e + 1) + " references out-of-range node " +
                                      std::to_string(el[a] + 1));
        double* G = pre.shape_gradients.data() + (size_t)e * 3 * nn;
        if (mesh.kind == ElementKind::T4) {
            Mat3 J;  // columns x2-x1, x3-x1, x4-x1
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) J.m[i][j] = mesh.nodes[el[j + 1]][i] - mesh.nodes[el[0]][i];
            const double dJ = det(J);
            const double V = dJ / 6.0;
            if (!(V > 0)) throw ValidationError("degenerate or inverted element " + std::to_string(e + 1));
            pre.ref_volume[e] = V;
            const Mat3 JinvT = transpose(inverse(J));
            for (int a = 0; a < 4; ++a)
                for (int i = 0; i < 3; ++i)
                    G[a * 3 + i] = JinvT.m[i][0] * kT4Xi[a][0] + JinvT.m[i][1] * kT4Xi[a][1] +
                                   JinvT.m[i][2] * kT4Xi[a][2];
        } else {
            Mat3 J0;  // dX/dxi at the centroid = X Xi^T / 8
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double s = 0;
                    for (int a = 0; a < 8; ++a) s += mesh.nodes[el[a]][i] * kH8Sign[a][j];
                    J0.m[i][j] = s / 8.0;
                }
            const double dJ = det(J0);
            if (!(dJ > 0)) throw ValidationError("degenerate or inverted element " + std::to_string(e + 1));
            pre.det_jacobian[e] = dJ;
            pre.ref_volume[e] = 8.0 * dJ;  // mesh.hpp:44
            const Mat3 JinvT = transpose(inverse(J0));
            for (int a = 0; a < 8; ++a)
                for (int i = 0; i < 3; ++i)
                    G[a * 3 + i] = (JinvT.m[i][0] * kH8Sign[a][0] + JinvT.m[i][1] * kH8Sign[a][1] +
                                    JinvT.m[i][2] * kH8Sign[a][2]) / 8.0;
            double X[24];
            for (int a = 0; a < 8; ++a)
                for (int i = 0; i < 3; ++i) X[a * 3 + i] = mesh.nodes[el[a]][i];
            hourglass_basis_for_element(X, G, pre.hourglass_basis.data() + (size_t)e * 32);
        }
    }
    // Adjacency CSR: ascending element, then local index (mesh.hpp:58-61).
    pre.adjacency_offsets.assign(N + 1, 0);
    for (int e = 0; e < E; ++e)
        for (int a = 0; a < nn; ++a) pre.adjacency_offsets[mesh.elements[e][a] + 1]++;
    for (int i = 0; i < N; ++i) pre.adjacency_offsets[i + 1] += pre.adjacency_offsets[i];
    pre.adjacency.assign((size_t)E * nn, {0, 0});
    std::vector<int> fill(pre.adjacency_offsets.begin(), pre.adjacency_offsets.end() - 1);
    for (int e = 0; e < E; ++e)
        for (int a = 0; a < nn; ++a) pre.adjacency[fill[mesh.elements[e][a]]++] = {e, a};
    // Equal-split lumping, accumulated in adjacency order.
    pre.lumped_mass.assign(N, 0.0);
    pre.lumped_heat_capacity_ref.assign(N, 0.0);
    pre.node_volume.assign(N, 0.0);
    for (int i = 0; i < N; ++i)
        for (int k = pre.adjacency_offsets[i]; k < pre.adjacency_offsets[i + 1]; ++k) {
            const double V = pre.ref_volume[pre.adjacency[k].first];
            pre.lumped_mass[i] += density * V / nn;
            pre.lumped_heat_capacity_ref[i] += density * ref_specific_heat * V / nn;
            pre.node_volume[i] += V / nn;
        }
    return pre;
}

double min_edge_length(const Mesh& mesh, int e) {
    static const int t4e[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    static const int h8e[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                   {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    const auto& el = mesh.elements[e];
    const bool t4 = mesh.kind == ElementKind::T4;
    const int ne = t4 ? 6 : 12;
    double L = std::numeric_limits<double>::infinity();
    for (int k = 0; k < ne; ++k) {
        const int a = t4 ? t4e[k][0] : h8e[k][0], b = t4 ? t4e[k][1] : h8e[k][1];
        double d2 = 0;
        for (int i = 0; i < 3; ++i) {
            const double d = mesh.nodes[el[a]][i] - mesh.nodes[el[b]][i];
            d2 += d * d;
        }
        L = std::min(L, std::sqrt(d2));
    }
    return L;
}

// mesh.hpp:92-97.
CriticalTimestep critical_timestep(const Mesh& mesh, const MaterialModel& m) {
    const double rho = m.thermal.density;
    const double cd = std::sqrt((m.hyperelastic.kappa + 4.0 * m.hyperelastic.mu / 3.0) / rho);
    const double cmin = m.thermal.specific_heat.min_value();
    const double kmax = m.thermal.conductivity.max_eigenvalue();
    double Lmin = std::numeric_limits<double>::infinity();
    for (int e = 0; e < mesh.element_count(); ++e) Lmin = std::min(Lmin, min_edge_length(mesh, e));
    CriticalTimestep ct;
    ct.mechanical = 0.9 * Lmin / cd;
    ct.thermal = 0.9 * (rho * cmin * Lmin * Lmin) / (2.0 * kmax * 3.0);
    return ct;
}

// ============================================================ materials (materials.hpp:13-133)
PronySeries PronySeries::from_terms(std::vector<PronyTerm> terms) {
    double s = 0;
    for (const auto& t : terms) {
        if (!(t.phi > 0) || !(t.tau > 0)) throw ValidationError("Prony terms need phi > 0 and tau > 0");
        s += t.phi;
    }
    if (!(s < 1.0)) throw ValidationError("Prony weights must sum to < 1");
    PronySeries p;
    p.terms = std::move(terms);
    p.phi_inf = 1.0 - s;
    return p;
}

// Clamped piecewise-linear interpolation.
static double interp_pairs(const std::vector<std::pair<double, double>>& t, double T) {
    if (t.empty()) throw ValidationError("empty property table");
    if (t.size() == 1 || T <= t.front().first) return t.front().second;
    if (T >= t.back().first) return t.back().second;
    size_t j = 0;
    while (j + 2 < t.size() && T >= t[j + 1].first) ++j;
    const double w = (T - t[j].first) / (t[j + 1].first - t[j].first);
    return t[j].second + (t[j + 1].second - t[j].second) * w;
}
double ScalarTable::at(double T) const { return interp_pairs(entries, T); }
double ScalarTable::min_value() const {
    double v = std::numeric_limits<double>::infinity();
    for (auto& e : entries) v = std::min(v, e.second);
    return v;
}
double ScalarTable::max_value() const {
    double v = -std::numeric_limits<double>::infinity();
    for (auto& e : entries) v = std::max(v, e.second);
    return v;
}
double interp_property(const ScalarTable& table, double T) { return table.at(T); }

Mat3 ConductivityTable::at(double T) const {
    if (entries.empty()) throw ValidationError("empty conductivity table");
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            std::vector<std::pair<double, double>> t;
            for (auto& e : entries) t.push_back({e.temperature, e.tensor.m[i][j]});
            r.m[i][j] = interp_pairs(t, T);
        }
    return r;
}
double ConductivityTable::max_eigenvalue() const {
    double v = -std::numeric_limits<double>::infinity();
    for (auto& e : entries) v = std::max(v, sym_max_eigenvalue(e.tensor));
    return v;
}

// materials.hpp:99-102; Table 5 energy.
double strain_energy(const Mat3& C, const HyperelasticParams& p, const Vec3* fiber) {
    const double dC = det(C);
    if (!(dC > 0)) throw ValidationError("non-SPD C");
    const double J = std::sqrt(dC);
    const double Jm23 = std::pow(J, -2.0 / 3.0);
    const double I1b = Jm23 * trace(C);
    double psi = 0.5 * p.mu * (I1b - 3.0) + 0.5 * p.kappa * (J - 1.0) * (J - 1.0);
    if (p.eta_a > 0) {
        if (!fiber) throw ValidationError("fiber required when eta_a > 0");
        const Vec3 Ca = C * (*fiber);
        const double I4b = Jm23 * ((*fiber)[0] * Ca[0] + (*fiber)[1] * Ca[1] + (*fiber)[2] * Ca[2]);
        psi += 0.5 * p.eta_a * (I4b - 1.0) * (I4b - 1.0);
    }
    return psi;
}

// materials.hpp:104-106: S = 2 dPsi/dC (checked against FD in tests).
// Non-throwing core: a non-SPD (or non-finite) C yields NaN and sets *bad, which
// the engine turns into a ValidationError after completing the step (C25).
//
// Evaluated from the strain X = C - I rather than from C: with soft tissue near
// its reference state (strains 1e-6..1e-2) every O(1) difference in the textbook
// form (I - I1/3 C^-1, J - 1, I4b - 1) loses ~|log10 strain| digits, and those
// rounding errors, not the physics, would then dominate an fp64 comparison of two
// implementations.  The identities used are exact:
//   det C - 1 = tr X + (tr^2 X - tr X^2)/2 + det X,
//   I - (I1/3) C^-1 = C^-1 dev(X),   J - 1 = (det C - 1)/(J + 1),
//   J^-2/3 - 1 = -(det C - 1) / (c (c^2 + c + 1)),  c = (det C)^(1/3).
static Mat3 pk2_from_strain(const Mat3& X, const HyperelasticParams& p, const Vec3* fiber, bool* bad) {
    const double i1 = trace(X);
    const double i2 = 0.5 * (i1 * i1 - trace(X * X));
    const double d1 = i1 + i2 + det(X);  // det C - 1
    if (!(d1 > -1.0)) {
        *bad = true;
        Mat3 r;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) r.m[i][j] = std::numeric_limits<double>::quiet_NaN();
        return r;
    }
    const double J = std::sqrt(1.0 + d1);
    const double Jm1 = d1 / (J + 1.0);
    const double c = std::cbrt(1.0 + d1);
    const double Jm23m1 = -d1 / (c * (c * c + c + 1.0));
    const double Jm23 = 1.0 + Jm23m1;
    const Mat3 Ci = inverse(Mat3::identity() + X);
    const Mat3 M = Ci * (X - (i1 / 3.0) * Mat3::identity());
    Mat3 S = (0.5 * p.mu * Jm23) * (M + transpose(M));
    if (p.eta_a > 0) {
        if (!fiber) throw ValidationError("fiber required when eta_a > 0");
        const Vec3& a = *fiber;
        const Vec3 Xa = X * a;
        const double aa = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
        const double aXa = a[0] * Xa[0] + a[1] * Xa[1] + a[2] * Xa[2];
        const double I4 = aa + aXa;
        const double I4bm1 = Jm23m1 + Jm23 * ((aa - 1.0) + aXa);  // J^-2/3 I4 - 1
        S = S + (2.0 * p.eta_a * I4bm1 * Jm23) * (outer(a, a) - (I4 / 3.0) * Ci);
    }
    S = S + (p.kappa * J * Jm1) * Ci;
    return S;
}
static Mat3 pk2_core(const Mat3& C, const HyperelasticParams& p, const Vec3* fiber, bool* bad) {
    return pk2_from_strain(C - Mat3::identity(), p, fiber, bad);
}
Mat3 pk2_stress(const Mat3& C, const HyperelasticParams& p, const Vec3* fiber) {
    bool bad = false;
    Mat3 S = pk2_core(C, p, fiber, &bad);
    if (bad) throw ValidationError("non-SPD C");
    return S;
}

// materials.hpp:108-114; Eq. 11.  F_ther - I, formed from the
// stretch increments alpha dT directly (see pk2_from_strain on why not 1 + alpha dT - 1).
static Mat3 thermal_deformation_delta(double T, const ExpansionSpec& s, const Vec3& m, const Vec3& n) {
    auto dot = [](const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
    const double dT = T - s.reference_temperature;
    const double ei = s.alpha_i * dT;
    Mat3 D = ei * Mat3::identity();
    if (s.kind != ExpansionKind::Isotropic) {
        if (std::fabs(dot(m, m) - 1.0) > 1e-6) throw ValidationError("expansion axis m not unit");
        D = D + (s.alpha_m * dT - ei) * outer(m, m);
    }
    if (s.kind == ExpansionKind::Orthotropic) {
        if (std::fabs(dot(n, n) - 1.0) > 1e-6 || std::fabs(dot(m, n)) > 1e-6)
            throw ValidationError("expansion axes not orthonormal");
        D = D + (s.alpha_n * dT - ei) * outer(n, n);
    }
    return D;
}
Mat3 thermal_deformation_gradient(double T, const ExpansionSpec& s, const Vec3& m, const Vec3& n) {
    return Mat3::identity() + thermal_deformation_delta(T, s, m, n);
}

// materials.hpp:116-120; Eq. 8-10, from the displacement gradient
// Hd = F - I and Delta = F_ther - I:  F_elas - I = (Hd - Delta) F_ther^-1,
// C_elas - I = Hel + Hel^T + Hel^T Hel.
static Mat3 total_pk2_from_grad(const Mat3& Hd, const Mat3& Delta, const HyperelasticParams& p, const Vec3* fiber,
                                bool* bad) {
    const Mat3 Fth = Mat3::identity() + Delta;
    const Mat3 Fi = inverse(Fth);
    const Mat3 Hel = (Hd - Delta) * Fi;
    const Mat3 X = Hel + transpose(Hel) + transpose(Hel) * Hel;
    const Mat3 Sint = pk2_from_strain(X, p, fiber, bad);
    return det(Fth) * (Fi * Sint * transpose(Fi));
}
static Mat3 total_pk2_core(const Mat3& F, const Mat3& Fth, const HyperelasticParams& p, const Vec3* fiber,
                           bool* bad) {
    return total_pk2_from_grad(F - Mat3::identity(), Fth - Mat3::identity(), p, fiber, bad);
}
Mat3 total_pk2_stress(const Mat3& F, const Mat3& Fth, const HyperelasticParams& p, const Vec3* fiber) {
    bool bad = false;
    Mat3 S = total_pk2_core(F, Fth, p, fiber, &bad);
    if (bad) throw ValidationError("non-SPD C");
    return S;
}

// materials.hpp:122-127.
Mat3 prony_update(const Mat3& S, std::span<Mat3> history, double dt, const PronySeries& prony) {
    if (history.size() != prony.terms.size()) throw ValidationError("history length mismatch");
    Mat3 St = S;
    for (size_t i = 0; i < prony.terms.size(); ++i) {
        const double phi = prony.terms[i].phi, tau = prony.terms[i].tau;
        const double a = dt * phi / (dt + tau);
        const double b = tau / (dt + tau);
        history[i] = a * S + b * history[i];
        St = St - history[i];
    }
    return St;
}

double relaxation_function(double t, const PronySeries& prony) {
    double v = prony.phi_inf;
    for (const auto& term : prony.terms) v += term.phi * std::exp(-t / term.tau);
    return v;
}

// ============================================================ bioheat (bioheat.hpp:37-69)
template <int NN>
static std::array<double, NN> thermal_load_core(const Mat3& F, const double* grad, const Mat3& D, const double* Te,
                                                double V, bool* bad) {
    // Dense Eq. 18/19 assembly: K = V det(F) B^T D B with B = F^-T G (3 x NN).
    const Mat3 FiT = transpose(inverse_core(F, bad));
    const double dF = det(F);
    double B[3][NN];
    for (int a = 0; a < NN; ++a)
        for (int i = 0; i < 3; ++i)
            B[i][a] = FiT.m[i][0] * grad[a * 3 + 0] + FiT.m[i][1] * grad[a * 3 + 1] + FiT.m[i][2] * grad[a * 3 + 2];
    std::array<double, NN> f{};
    for (int a = 0; a < NN; ++a) {
        double fa = 0;
        for (int b = 0; b < NN; ++b) {
            double k = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) k += B[i][a] * D.m[i][j] * B[j][b];
            fa += V * dF * k * Te[b];
        }
        f[a] = fa;
    }
    return f;
}
template <int NN>
std::array<double, NN> element_thermal_load(const Mat3& F, const double* grad, const Mat3& D, const double* Te,
                                            double V) {
    bool bad = false;
    auto f = thermal_load_core<NN>(F, grad, D, Te, V, &bad);
    if (bad) throw ValidationError("singular F");
    return f;
}
template std::array<double, 4> element_thermal_load<4>(const Mat3&, const double*, const Mat3&, const double*, double);
template std::array<double, 8> element_thermal_load<8>(const Mat3&, const double*, const Mat3&, const double*, double);

// bioheat.hpp:49-63; Eq. 20.
void step_temperature(ThermalState& st, std::span<const double> f, std::span<const double> Qr,
                      const ThermalProps& p, std::span<const double> Vn, const ThermalBCs& bcs,
                      double dt, bool td, double fixed_T) {
    const int N = (int)st.temperatures.size();
    for (int i = 0; i < N; ++i) {
        const double T = st.temperatures[i];
        const double c = p.specific_heat.at(td ? T : fixed_T);
        const double C = p.density * c * Vn[i];
        if (C <= 0) throw ValidationError("nonpositive C_diag at node " + std::to_string(i));
        const double rhs = -f[i] - p.perfusion_rate * p.blood_specific_heat * Vn[i] * (T - p.arterial_temperature) +
                           p.metabolic_rate * Vn[i] + Qr[i];
        st.temperatures[i] = T + dt / C * rhs;
    }
    for (const auto& [node, value] : bcs.fixed) st.temperatures[node] = value;
}

// bioheat.hpp:65-69: lump active regional sources by element volume shares.
void accumulate_nodal_sources(std::vector<double>& power, const HeatSourceSet& sources, const Mesh& mesh,
                              const PrecomputedMesh& pre, double time) {
    std::fill(power.begin(), power.end(), 0.0);
    const int nn = pre.nodes_per_elem();
    for (const auto& r : sources.regional) {
        if (!r.active_at(time)) continue;
        for (int e : r.elements)
            for (int a = 0; a < nn; ++a) power[mesh.elements[e][a]] += r.q_r * pre.ref_volume[e] / nn;
    }
}

// ============================================================ mechanics (mechanics.hpp:15-110)
MechState MechState::zero(int N, int E, int P) {
    MechState s;
    s.disp.assign((size_t)3 * N, 0.0);
    s.disp_prev.assign((size_t)3 * N, 0.0);
    s.viscous.assign((size_t)E * P, Mat3{});
    return s;
}

// mechanics.hpp:49-53; Eq. 17: F = I + U G^T.
template <int NN>
Mat3 deformation_gradient(const double* U, const double* G) {
    Mat3 F = Mat3::identity();
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int a = 0; a < NN; ++a) s += U[a * 3 + i] * G[a * 3 + j];
            F.m[i][j] += s;
        }
    return F;
}
template Mat3 deformation_gradient<4>(const double*, const double*);
template Mat3 deformation_gradient<8>(const double*, const double*);
// U G^T alone: the mechanics phase keeps F - I at full relative precision.
template <int NN>
static Mat3 displacement_gradient(const double* U, const double* G) {
    Mat3 H;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int a = 0; a < NN; ++a) s += U[a * 3 + i] * G[a * 3 + j];
            H.m[i][j] = s;
        }
    return H;
}

// mechanics.hpp:55-69; Eqs. 25/26/28.
template <int NN>
static void internal_force_core(const Mat3& Hd, const double* G, const HyperelasticParams& params,
                                const Vec3* fiber, const Mat3& Delta, std::span<Mat3> hist, double dt,
                                const PronySeries& prony, double V, double* out, Mat3* S_tilde_out, bool* bad) {
    const Mat3 S = total_pk2_from_grad(Hd, Delta, params, fiber, bad);
    const Mat3 St = prony.empty() ? S : prony_update(S, hist, dt, prony);
    if (S_tilde_out) *S_tilde_out = St;
    const Mat3 P = V * (St + Hd * St);  // V F S~ with F = I + Hd
    for (int a = 0; a < NN; ++a)
        for (int i = 0; i < 3; ++i)
            out[a * 3 + i] = P.m[i][0] * G[a * 3 + 0] + P.m[i][1] * G[a * 3 + 1] + P.m[i][2] * G[a * 3 + 2];
}
template <int NN>
void element_internal_force(const Mat3& F, const double* G, const HyperelasticParams& params, const Vec3* fiber,
                            const Mat3& Fth, std::span<Mat3> hist, double dt, const PronySeries& prony, double V,
                            double* out, Mat3* S_tilde_out) {
    bool bad = false;
    internal_force_core<NN>(F - Mat3::identity(), G, params, fiber, Fth - Mat3::identity(), hist, dt, prony, V, out,
                            S_tilde_out, &bad);
    if (bad) throw ValidationError("non-SPD C");
}
template void element_internal_force<4>(const Mat3&, const double*, const HyperelasticParams&, const Vec3*,
                                        const Mat3&, std::span<Mat3>, double, const PronySeries&, double, double*,
                                        Mat3*);
template void element_internal_force<8>(const Mat3&, const double*, const HyperelasticParams&, const Vec3*,
                                        const Mat3&, std::span<Mat3>, double, const PronySeries&, double, double*,
                                        Mat3*);

// mechanics.hpp:71-78: f = k U Gamma^T Gamma.
void hourglass_force(const double* U, const double* gamma, double k, double* out) {
    double q[4][3];
    for (int al = 0; al < 4; ++al)
        for (int i = 0; i < 3; ++i) {
            double s = 0;
            for (int b = 0; b < 8; ++b) s += U[b * 3 + i] * gamma[al * 8 + b];
            q[al][i] = s;
        }
    for (int a = 0; a < 8; ++a)
        for (int i = 0; i < 3; ++i) {
            double s = 0;
            for (int al = 0; al < 4; ++al) s += q[al][i] * gamma[al * 8 + a];
            out[a * 3 + i] = k * s;
        }
}

// mechanics.hpp:86-97; Eq. 22 header form.
void step_displacement(MechState& st, std::span<const double> f, const MechBCs& bcs,
                       std::span<const double> M, double gamma, double dt, double next_time) {
    const int N = (int)M.size();
    std::vector<double> up((size_t)3 * N);
    for (int i = 0; i < N; ++i) {
        const double m = M[i];
        if (!(m > 0)) throw ValidationError("nonpositive lumped mass at node " + std::to_string(i));
        const double D = gamma * m;
        const double a = D / (2.0 * dt), b = m / (dt * dt);
        for (int c = 0; c < 3; ++c) {
            const size_t k = (size_t)3 * i + c;
            const double R = bcs.external_force.empty() ? 0.0 : bcs.external_force[k];
            up[k] = (R - f[k] + 2.0 * b * st.disp[k] + (a - b) * st.disp_prev[k]) / (a + b);
        }
    }
    for (int n : bcs.fixed_nodes)
        for (int c = 0; c < 3; ++c) up[(size_t)3 * n + c] = 0.0;
    for (const auto& p : bcs.prescribed) {
        const double v = p.value_at(next_time);
        for (int n : p.nodes) up[(size_t)3 * n + p.component] = v;
    }
    if (bcs.motion_override)
        for (int n = 0; n < N; ++n)
            if (auto v = bcs.motion_override(n, next_time))
                for (int c = 0; c < 3; ++c) up[(size_t)3 * n + c] = (*v)[c];
    st.disp_prev.swap(st.disp);
    st.disp.swap(up);
}

// ============================================================ engine (engine.hpp:83-143)
Engine::Engine(const Mesh& mesh, const PrecomputedMesh& pre, const MaterialModel& material,
               const MechBCs& mech_bcs, const ThermalBCs& thermal_bcs, const HeatSourceSet& sources,
               const SimulationConfig& config)
    : mesh_(mesh), pre_(pre), material_(material), mech_bcs_(mech_bcs), thermal_bcs_(thermal_bcs),
      sources_(sources), config_(config) {
    if (!(config.dt > 0)) throw ValidationError("dt must be > 0");
    if (!config.allow_unstable_dt) {
        const CriticalTimestep ct = critical_timestep(mesh, material);
        if (config.dt > std::min(ct.thermal, ct.mechanical))
            throw ValidationError("dt above critical timestep");
    }
    if (material.hyperelastic.eta_a > 0 && !material.fiber && mesh.fiber_dirs.empty())
        throw ValidationError("eta_a > 0 requires a fiber direction");
    const int N = mesh.node_count(), E = mesh.element_count(), nn = mesh.nodes_per_elem();
    const int P = (int)material.prony.terms.size();
    state_.thermal.temperatures.assign(N, thermal_bcs.initial_temperature);
    state_.mech = MechState::zero(N, E, P);
    f_cache_.assign(E, Mat3::identity());
    f_ther_cache_.assign(E, Mat3::identity());
    f_ther_delta_.assign(E, Mat3{});
    stress_cache_.assign(E, Mat3{});
    element_thermal_loads_.assign((size_t)E * nn, 0.0);
    element_forces_.assign((size_t)E * 3 * nn, 0.0);
    assembled_load_.assign(N, 0.0);
    assembled_force_.assign((size_t)3 * N, 0.0);
    nodal_source_.assign(N, 0.0);
    external_force_total_.assign((size_t)3 * N, 0.0);
    for (int i = 0; i < N; ++i)
        for (int c = 0; c < 3; ++c) {
            const size_t k = (size_t)3 * i + c;
            const double ext = mech_bcs.external_force.empty() ? 0.0 : mech_bcs.external_force[k];
            external_force_total_[k] = ext + mech_bcs.body_force[c] * pre.node_volume[i];
        }
    mech_bcs_.external_force = external_force_total_;
    source_active_.assign(sources.regional.size(), 0);
#ifdef _OPENMP
    workers_ = config.workers > 0 ? config.workers : omp_get_max_threads();
#else
    workers_ = 1;
#endif
}

void Engine::set_nodal_source_override(const double* power) {
    if (power) {
        std::copy(power, power + nodal_source_.size(), nodal_source_.begin());
        source_override_ = true;
    } else {
        source_override_ = false;
        sources_initialized_ = false;
    }
}

void Engine::refresh_nodal_sources() {
    if (source_override_) return;
    bool changed = !sources_initialized_;
    for (size_t r = 0; r < sources_.regional.size(); ++r) {
        const char a = sources_.regional[r].active_at(state_.thermal.time) ? 1 : 0;
        if (a != source_active_[r]) changed = true;
        source_active_[r] = a;
    }
    if (changed) accumulate_nodal_sources(nodal_source_, sources_, mesh_, pre_, state_.thermal.time);
    sources_initialized_ = true;
}

template <int NN>
void Engine::thermal_element_phase(bool compute_f) {
    const int E = mesh_.element_count();
    const auto& T = state_.thermal.temperatures;
    const auto& u = state_.mech.disp;
    const bool td = config_.temperature_dependent;
    int bad_elem = E;
#pragma omp parallel for num_threads(workers_) schedule(static) reduction(min : bad_elem)
    for (int e = 0; e < E; ++e) {
        const auto& el = mesh_.elements[e];
        const double* G = pre_.gradients(e);
        if (compute_f) {
            double U[3 * NN];
            for (int a = 0; a < NN; ++a)
                for (int i = 0; i < 3; ++i) U[a * 3 + i] = u[(size_t)3 * el[a] + i];
            f_cache_[e] = deformation_gradient<NN>(U, G);
        }
        double Te[NN], Tsum = 0;
        for (int a = 0; a < NN; ++a) {
            Te[a] = T[el[a]];
            Tsum += Te[a];
        }
        const double Tbar = Tsum / NN;
        const Mat3 D = material_.thermal.conductivity.at(td ? Tbar : fixed_property_temperature_);
        bool bad = false;
        const auto f = thermal_load_core<NN>(f_cache_[e], G, D, Te, pre_.geometry_factor(e), &bad);
        if (bad) bad_elem = std::min(bad_elem, e);
        for (int a = 0; a < NN; ++a) element_thermal_loads_[(size_t)e * NN + a] = f[a];
    }
    if (bad_elem < E && (element_error_ < 0 || bad_elem < element_error_)) element_error_ = bad_elem;
}

void Engine::thermal_node_phase() {
    const int N = mesh_.node_count(), nn = mesh_.nodes_per_elem();
#pragma omp parallel for num_threads(workers_) schedule(static)
    for (int i = 0; i < N; ++i) {
        double s = 0;
        for (int k = pre_.adjacency_offsets[i]; k < pre_.adjacency_offsets[i + 1]; ++k) {
            const auto [e, a] = pre_.adjacency[k];
            s += element_thermal_loads_[(size_t)e * nn + a];
        }
        assembled_load_[i] = s;
    }
    step_temperature(state_.thermal, assembled_load_, nodal_source_, material_.thermal, pre_.node_volume,
                     thermal_bcs_, config_.dt, config_.temperature_dependent, fixed_property_temperature_);
}

template <int NN>
void Engine::mechanics_element_phase(bool compute_f) {
    const int E = mesh_.element_count();
    const int P = (int)material_.prony.terms.size();
    const auto& u = state_.mech.disp;
    const double kh = config_.hourglass_stiffness * material_.hyperelastic.mu;
    int bad_elem = E;
#pragma omp parallel for num_threads(workers_) schedule(static) reduction(min : bad_elem)
    for (int e = 0; e < E; ++e) {
        const auto& el = mesh_.elements[e];
        const double* G = pre_.gradients(e);
        double U[3 * NN];
        for (int a = 0; a < NN; ++a)
            for (int i = 0; i < 3; ++i) U[a * 3 + i] = u[(size_t)3 * el[a] + i];
        const Mat3 Hd = displacement_gradient<NN>(U, G);
        if (compute_f) f_cache_[e] = Mat3::identity() + Hd;
        const Vec3* fiber = nullptr;
        if (!mesh_.fiber_dirs.empty()) fiber = &mesh_.fiber_dirs[e];
        else if (material_.fiber) fiber = &*material_.fiber;
        double f[3 * NN];
        std::span<Mat3> hist(state_.mech.viscous.data() + (size_t)e * P, P);
        bool bad = false;
        internal_force_core<NN>(Hd, G, material_.hyperelastic, fiber, f_ther_delta_[e], hist, config_.dt,
                                material_.prony, pre_.geometry_factor(e), f, &stress_cache_[e], &bad);
        if (bad) bad_elem = std::min(bad_elem, e);
        if constexpr (NN == 8) {
            double fh[24];
            const double k = kh * std::cbrt(pre_.ref_volume[e]);
            hourglass_force(U, pre_.hourglass_basis.data() + (size_t)e * 32, k, fh);
            for (int q = 0; q < 24; ++q) f[q] += fh[q];
        }
        for (int q = 0; q < 3 * NN; ++q) element_forces_[(size_t)e * 3 * NN + q] = f[q];
    }
    if (bad_elem < E && (element_error_ < 0 || bad_elem < element_error_)) element_error_ = bad_elem;
}

void Engine::mechanics_node_phase() {
    const int N = mesh_.node_count(), nn = mesh_.nodes_per_elem();
#pragma omp parallel for num_threads(workers_) schedule(static)
    for (int i = 0; i < N; ++i) {
        double s[3] = {0, 0, 0};
        for (int k = pre_.adjacency_offsets[i]; k < pre_.adjacency_offsets[i + 1]; ++k) {
            const auto [e, a] = pre_.adjacency[k];
            for (int c = 0; c < 3; ++c) s[c] += element_forces_[(size_t)e * 3 * nn + a * 3 + c];
        }
        for (int c = 0; c < 3; ++c) assembled_force_[(size_t)3 * i + c] = s[c];
    }
    step_displacement(state_.mech, assembled_force_, mech_bcs_, pre_.lumped_mass, config_.damping_gamma,
                      config_.dt, state_.thermal.time + config_.dt);
}

void Engine::check_finite(std::span<const double> v, const char* field, int stride) const {
    for (size_t k = 0; k < v.size(); ++k)
        if (!std::isfinite(v[k])) {
            const int node = (int)(k / stride);
            throw InstabilityError(std::string("non-finite ") + field + " at step " + std::to_string(state_.step) +
                                       ", node " + std::to_string(node),
                                   state_.step, node);
        }
}

template <int NN>
void Engine::step_impl() {
    const bool coupled = config_.mode == CouplingMode::Coupled;
    if (config_.mode != CouplingMode::MechanicalOnly) {
        thermal_element_phase<NN>(true);
        refresh_nodal_sources();
        thermal_node_phase();
    }
    if (config_.mode != CouplingMode::ThermalOnly) {
        const int E = mesh_.element_count();
        const bool exp = coupled && config_.expansion_enabled && material_.expansion.has_value();
        if (exp) {
            const auto& T = state_.thermal.temperatures;
#pragma omp parallel for num_threads(workers_) schedule(static)
            for (int e = 0; e < E; ++e) {
                double Ts = 0;
                for (int a = 0; a < NN; ++a) Ts += T[mesh_.elements[e][a]];
                const double Tbar = Ts / NN;
                const Vec3& m = mesh_.expansion_axes.empty() ? material_.axis_m : mesh_.expansion_axes[e][0];
                const Vec3& n = mesh_.expansion_axes.empty() ? material_.axis_n : mesh_.expansion_axes[e][1];
                f_ther_delta_[e] = thermal_deformation_delta(Tbar, *material_.expansion, m, n);
                f_ther_cache_[e] = Mat3::identity() + f_ther_delta_[e];
            }
        }
        mechanics_element_phase<NN>(!coupled);
        mechanics_node_phase();
    }
    // The step completes before reporting (the GPU cannot abort mid-kernel; C25):
    // element-kernel errors first (they occur earlier in the step), then non-finite state.
    if (element_error_ >= 0) {
        const int e = element_error_;
        element_error_ = -1;
        throw ElementError("non-SPD C or singular F in element " + std::to_string(e) + " at step " +
                               std::to_string(state_.step),
                           state_.step, e);
    }
    check_finite(state_.thermal.temperatures, "temperature", 1);
    check_finite(state_.mech.disp, "displacement", 3);
    state_.thermal.time += config_.dt;
    state_.step += 1;
}

void Engine::step() {
    if (mesh_.kind == ElementKind::T4) step_impl<4>();
    else step_impl<8>();
}

// engine.hpp:107-108: kinetic (backward-difference velocity) + hyperelastic strain energy.
double Engine::total_energy() const {
    const int N = mesh_.node_count(), E = mesh_.element_count(), nn = mesh_.nodes_per_elem();
    double Ek = 0;
    for (int i = 0; i < N; ++i)
        for (int c = 0; c < 3; ++c) {
            const size_t k = (size_t)3 * i + c;
            const double v = (state_.mech.disp[k] - state_.mech.disp_prev[k]) / config_.dt;
            Ek += 0.5 * pre_.lumped_mass[i] * v * v;
        }
    double Es = 0;
    for (int e = 0; e < E; ++e) {
        double U[24];
        for (int a = 0; a < nn; ++a)
            for (int i = 0; i < 3; ++i) U[a * 3 + i] = state_.mech.disp[(size_t)3 * mesh_.elements[e][a] + i];
        const Mat3 F = nn == 4 ? deformation_gradient<4>(U, pre_.gradients(e)) : deformation_gradient<8>(U, pre_.gradients(e));
        const Mat3 Fi = inverse(f_ther_cache_[e]);
        const Mat3 Fel = F * Fi;
        const Vec3* fiber = !mesh_.fiber_dirs.empty() ? &mesh_.fiber_dirs[e] : (material_.fiber ? &*material_.fiber : nullptr);
        Es += pre_.ref_volume[e] * det(f_ther_cache_[e]) * strain_energy(transpose(Fel) * Fel, material_.hyperelastic, fiber);
    }
    return Ek + Es;
}

// ---- ablation_volume ----
// k = #nodes at or above the threshold.  With t_ij = (T_i - thr) / (T_i - T_j) the
// fraction of edge i -> j above the threshold (i above, j below):
//   k = 1 (node a):      t_ab t_ac t_ad                      (corner tetrahedron)
//   k = 3 (node d below): 1 - s_da s_db s_dc,  s_dj = (thr - T_d) / (T_j - T_d)
//   k = 2 (a, b above):  the wedge a p_ac p_ad | b p_bc p_bd split into the tetrahedra
//                        (a p_ac p_ad p_bd), (a p_ac p_bc p_bd), (a b p_bc p_bd), whose
//                        barycentric determinants give
//                        t_ac t_ad (1 - t_bd) + t_ac t_bd (1 - t_bc) + t_bc t_bd.
double tet_fraction_above(const double T[4], double thr) {
    int up[4], dn[4], nu = 0, nd = 0;
    for (int i = 0; i < 4; ++i) {
        if (T[i] >= thr) up[nu++] = i;
        else dn[nd++] = i;
    }
    auto t = [&](int i, int j) { return (T[i] - thr) / (T[i] - T[j]); };
    switch (nu) {
        case 0: return 0.0;
        case 4: return 1.0;
        case 1: return t(up[0], dn[0]) * t(up[0], dn[1]) * t(up[0], dn[2]);
        case 3: {
            const int d = dn[0];
            auto s = [&](int j) { return (thr - T[d]) / (T[j] - T[d]); };
            return 1.0 - s(up[0]) * s(up[1]) * s(up[2]);
        }
        default: {
            const int a = up[0], b = up[1], c = dn[0], d = dn[1];
            const double tac = t(a, c), tad = t(a, d), tbc = t(b, c), tbd = t(b, d);
            return tac * tad * (1.0 - tbd) + tac * tbd * (1.0 - tbc) + tbc * tbd;
        }
    }
}

namespace {
const int kHexTets[6][4] = {{0, 1, 2, 6}, {0, 2, 3, 6}, {0, 3, 7, 6}, {0, 7, 4, 6}, {0, 4, 5, 6}, {0, 5, 1, 6}};
}

AblationReport ablation_volume(const Mesh& mesh, std::span<const double> T, double threshold,
                               const std::vector<double>* disp) {
    AblationReport r;
    const int nn = mesh.nodes_per_elem();
    const int ntet = nn == 4 ? 1 : 6;
    for (int e = 0; e < mesh.element_count(); ++e) {
        double ve = 0;
        for (int k = 0; k < ntet; ++k) {
            int id[4];
            for (int q = 0; q < 4; ++q) id[q] = mesh.elements[e][nn == 4 ? q : kHexTets[k][q]];
            Vec3 x[4];
            double Tv[4];
            for (int q = 0; q < 4; ++q) {
                x[q] = mesh.nodes[id[q]];
                if (disp)
                    for (int c = 0; c < 3; ++c) x[q][c] += (*disp)[3 * (size_t)id[q] + c];
                Tv[q] = T[id[q]];
            }
            const double f = tet_fraction_above(Tv, threshold);
            if (f == 0.0) continue;
            Mat3 M;
            for (int c = 0; c < 3; ++c)
                for (int q = 0; q < 3; ++q) M[c][q] = x[q + 1][c] - x[0][c];
            ve += f * std::fabs(det(M)) / 6.0;
        }
        if (ve > 0) {
            r.volume += ve;
            ++r.elements_above;
        }
    }
    return r;
}

}  // namespace tve_oracle
