// lp_oracle.cpp -- plain, slow, obviously-correct CPU oracle for the Lightplane
// Renderer (Cao et al., arXiv 2404.19760). TEST INFRASTRUCTURE ONLY: it may be
// loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs, never by the product path. It shares no code, header
// or constant with paper_2404_19760_b200/ (the CUDA path).
//
// Everything is fp64. One ray at a time, rays in index order, gradient sums in
// ray order. The forward is the "store-all" (naive) evaluation of Eq. 1 that
// the paper's fused kernel avoids, and the backward is the
// hand-derived reverse mode over the stored per-sample values (Eq. 3, P:337-348,
// extended by the background and tau terms, readings R5, R12).
//
// Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
//
// Parity pins: every function below is pinned by tests/test_oracle_*.py
// (closed forms, special cases, adjointness, finite differences, literal
// O(S^2) derivative, invariants). None is "parity unpinned".
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

struct Field {
  int kind;        // 0 = triplane, 1 = voxel
  int H, W, D, K;  // resolution along x, y, z; channels
  const double* plane[3];
  int n_layers;    // number of Linear layers
  const int* widths;   // n_layers + 1 entries
  const double* params;  // W_0[w1][w0], b_0[w1], W_1[w2][w1], b_1[w2], ...
  int contraction;     // 0 none, 1 per-axis, 2 radial (see contract())
  double contract_a;   // scale a
  int dir_freqs;       // F > 0: view-dependent field, two networks (see split_nets())
  int wsig[10], wcol[10];  // widths of g_sigma / g_v when dir_freqs > 0
};

struct Tap {
  int plane;
  int64_t cell;    // index of the K-vector within its plane / volume
  double w;
};

// Scene contraction (Supp. Eq. "contract"):
//   CC(x) = 0.5 * a x                                    if ||x|| <= 1
//   CC(x) = 0.5 * ((2 - a)(1 - 1/||x||) + a) (x/||x||)   if ||x|| > 1
// "We convert X, Y, Z axes into contract coordinates independently":
// mode 1 applies the formula to each coordinate with ||x|| = |x_k| (reading
// R25); mode 2 is the displayed Euclidean form. The contracted point is what
// the hashing scheme samples; Delta stays the world distance (reading R25).
double contract_1d(double x, double a) {
  double n = std::fabs(x);
  if (n <= 1.0) return 0.5 * (a * x);
  return 0.5 * (((2.0 - a) * (1.0 - 1.0 / n) + a) * (x / n));
}

void contract(const Field& F, double x[3]) {
  if (F.contraction == 1) {
    for (int k = 0; k < 3; ++k) x[k] = contract_1d(x[k], F.contract_a);
  } else if (F.contraction == 2) {
    double n = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
    const double a = F.contract_a;
    if (n <= 1.0) {
      for (int k = 0; k < 3; ++k) x[k] = 0.5 * (a * x[k]);
    } else {
      double s = (2.0 - a) * (1.0 - 1.0 / n) + a;
      for (int k = 0; k < 3; ++k) x[k] = 0.5 * (s * (x[k] / n));
    }
  }
}

// O1: hashing scheme h (P:202 trilinear on voxels; P:207-210 bilinear on the
// (x,y), (y,z), (z,x) planes, summed). World cube [-1,1]^3 -> index space
// [0, N-1] per axis (reading R8); a point with any |x_a| > 1 samples zero and
// has no taps (reading R11).
void axis(double x, int N, int* i, double* f) {
  double u = (x + 1.0) * 0.5 * (double)(N - 1);
  int ii = (int)std::floor(u);
  if (ii > N - 2) ii = N - 2;
  if (ii < 0) ii = 0;
  *i = ii;
  *f = u - (double)ii;
}

void sample_taps(const Field& F, const double x[3], std::vector<Tap>& taps) {
  taps.clear();
  if (std::fabs(x[0]) > 1.0 || std::fabs(x[1]) > 1.0 || std::fabs(x[2]) > 1.0) return;
  int ix, iy, iz;
  double fx, fy, fz;
  axis(x[0], F.H, &ix, &fx);
  axis(x[1], F.W, &iy, &fy);
  axis(x[2], F.D, &iz, &fz);
  if (F.kind == 1) {
    for (int dx = 0; dx < 2; ++dx)
      for (int dy = 0; dy < 2; ++dy)
        for (int dz = 0; dz < 2; ++dz) {
          double w = (dx ? fx : 1.0 - fx) * (dy ? fy : 1.0 - fy) * (dz ? fz : 1.0 - fz);
          int64_t cell = ((int64_t)(ix + dx) * F.W + (iy + dy)) * F.D + (iz + dz);
          taps.push_back({0, cell, w});
        }
  } else {
    // plane 0: xy, [H][W]; plane 1: yz, [W][D]; plane 2: zx, [D][H]
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        taps.push_back({0, (int64_t)(ix + a) * F.W + (iy + b), (a ? fx : 1 - fx) * (b ? fy : 1 - fy)});
      }
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        taps.push_back({1, (int64_t)(iy + a) * F.D + (iz + b), (a ? fy : 1 - fy) * (b ? fz : 1 - fz)});
      }
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        taps.push_back({2, (int64_t)(iz + a) * F.H + (ix + b), (a ? fz : 1 - fz) * (b ? fx : 1 - fx)});
      }
  }
}

void gather(const Field& F, const std::vector<Tap>& taps, double* h) {
  for (int k = 0; k < F.K; ++k) h[k] = 0.0;
  for (const Tap& t : taps) {
    const double* v = F.plane[t.plane] + t.cell * F.K;
    for (int k = 0; k < F.K; ++k) h[k] += t.w * v[k];
  }
}

void scatter(const Field& F, const std::vector<Tap>& taps, const double* dh, double* const* grad) {
  for (const Tap& t : taps) {
    double* g = grad[t.plane] + t.cell * F.K;
    for (int k = 0; k < F.K; ++k) g[k] += t.w * dh[k];
  }
}

// O2: the tiny MLP g, one network K -> H ... -> 1 + C (reading R6):
// z_l = W_l a_{l-1} + b_l, ReLU on hidden layers, identity on the last.
// zs[l] holds z_{l}, as[l] holds a_l (as[0] = input).
struct MlpTrace {
  std::vector<std::vector<double>> z, a;
};

void mlp_forward(const Field& F, const double* in, MlpTrace& tr) {
  const int L = F.n_layers;
  tr.z.assign(L, {});
  tr.a.assign(L + 1, {});
  tr.a[0].assign(in, in + F.widths[0]);
  const double* p = F.params;
  for (int l = 0; l < L; ++l) {
    int fin = F.widths[l], fout = F.widths[l + 1];
    const double* Wl = p;
    const double* bl = p + (int64_t)fout * fin;
    p = bl + fout;
    tr.z[l].assign(fout, 0.0);
    for (int i = 0; i < fout; ++i) {
      double s = bl[i];
      for (int k = 0; k < fin; ++k) s += Wl[(int64_t)i * fin + k] * tr.a[l][k];
      tr.z[l][i] = s;
    }
    tr.a[l + 1] = tr.z[l];
    if (l < L - 1)
      for (double& v : tr.a[l + 1]) v = v > 0.0 ? v : 0.0;
  }
}

// Reverse mode through the MLP: given dL/d(output z_{L-1}), accumulate
// parameter gradients and return dL/d(input).
void mlp_backward(const Field& F, const MlpTrace& tr, const double* dout, double* grad_params, double* din) {
  const int L = F.n_layers;
  std::vector<int64_t> off(L);
  int64_t o = 0;
  for (int l = 0; l < L; ++l) {
    off[l] = o;
    o += (int64_t)F.widths[l + 1] * F.widths[l] + F.widths[l + 1];
  }
  std::vector<double> delta(dout, dout + F.widths[L]);
  for (int l = L - 1; l >= 0; --l) {
    int fin = F.widths[l], fout = F.widths[l + 1];
    const double* Wl = F.params + off[l];
    double* gW = grad_params + off[l];
    double* gb = gW + (int64_t)fout * fin;
    for (int i = 0; i < fout; ++i) {
      gb[i] += delta[i];
      for (int k = 0; k < fin; ++k) gW[(int64_t)i * fin + k] += delta[i] * tr.a[l][k];
    }
    std::vector<double> prev(fin, 0.0);
    for (int k = 0; k < fin; ++k) {
      double s = 0.0;
      for (int i = 0; i < fout; ++i) s += Wl[(int64_t)i * fin + k] * delta[i];
      prev[k] = s;
    }
    if (l > 0)  // through the ReLU of layer l-1 (ReLU'(0) = 0)
      for (int k = 0; k < fin; ++k) prev[k] = tr.z[l - 1][k] > 0.0 ? prev[k] : 0.0;
    delta.swap(prev);
  }
  for (int k = 0; k < F.widths[0]; ++k) din[k] = delta[k];
}

// O3: heads (reading R7): sigma = softplus(o_0), c_k = sigmoid(o_k).
double softplus(double x) { return (x > 0.0 ? x : 0.0) + std::log1p(std::exp(-std::fabs(x))); }
double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

// View-dependent colour ("f_v(x_ij) is calculated by another MLP g_v
// taking the sampled feature and view directions as inputs"; reading R29).
// direnc(d) = for each axis k, for each frequency f = 2^0 .. 2^{F-1}:
// (sin(pi f d_k), cos(pi f d_k)), E = 6F values (F = 4 by default).
void direnc(const double* d, int F, double* e) {
  const double pi = 3.14159265358979323846;
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < F; ++i) {
      double a = pi * std::ldexp(1.0, i) * d[k];
      e[2 * (k * F + i)] = std::sin(a);
      e[2 * (k * F + i) + 1] = std::cos(a);
    }
}

// With dir_freqs = F > 0 the field's parameters hold two networks with the
// hidden widths of `widths` (reading R29): g_sigma: K -> hidden... -> 1 (the
// density logit) followed by g_v: K + 6F -> hidden... -> C (the colour logits),
// each packed W_0, b_0, W_1, b_1, ... like a single network.
int64_t net_params(int n_layers, const int* w) {
  int64_t n = 0;
  for (int l = 0; l < n_layers; ++l) n += (int64_t)w[l + 1] * w[l] + w[l + 1];
  return n;
}

void split_nets(const Field& F, Field& Fs, Field& Fv) {
  Fs = F;
  Fv = F;
  const int L = F.n_layers, C = F.widths[L] - 1;
  for (int l = 0; l <= L; ++l) {
    Fs.wsig[l] = F.widths[l];
    Fv.wcol[l] = F.widths[l];
  }
  Fs.wsig[L] = 1;
  Fv.wcol[0] = F.K + 6 * F.dir_freqs;
  Fv.wcol[L] = C;
  Fs.widths = Fs.wsig;
  Fv.widths = Fv.wcol;
  Fv.params = F.params + net_params(L, Fs.widths);
}

// Everything stored for one ray by the store-all forward.
struct RayTrace {
  int S;
  double delta;
  std::vector<std::vector<Tap>> taps;
  std::vector<MlpTrace> mlp;
  std::vector<MlpTrace> mlpv;             // g_v traces (view-dependent fields)
  std::vector<double> e;                  // direnc(d) of the ray
  std::vector<double> t;                  // t_j = near + j Delta (ray parameter of sample j)
  std::vector<double> sigma, tau, T, w;   // tau_j = sum_{n<=j} Delta sigma_n, T_j = exp(-tau_j)
  std::vector<std::vector<double>> c;     // colours c_j (C each)
};

// O4: store-all forward of Eq. 1 for ray r.
// x_j = o + (near + j Delta) d, Delta = max(far - near, 0)/R, j = 0..R (P:234,
// P:247; reading R2). Weights w_0 = 0 and, for j >= 1,
// w_j = T_{j-1} - T_j evaluated as e^{-tau_{j-1}} (-expm1(-Delta sigma_j))
// (reading R13; the same number, without the cancellation).
void trace_ray(const Field& F, const double* o, const double* d, double nearv, double farv, int S,
               RayTrace& rt) {
  const int C = F.widths[F.n_layers] - 1;
  const int R = S - 1;
  rt.S = S;
  double span = farv - nearv;
  rt.delta = (span > 0.0 ? span : 0.0) / (double)R;
  rt.taps.assign(S, {});
  rt.mlp.assign(S, {});
  rt.mlpv.assign(F.dir_freqs > 0 ? S : 0, {});
  rt.t.assign(S, 0.0);
  rt.sigma.assign(S, 0.0);
  rt.tau.assign(S, 0.0);
  rt.T.assign(S, 0.0);
  rt.w.assign(S, 0.0);
  rt.c.assign(S, std::vector<double>(C, 0.0));
  std::vector<double> h(F.K);
  Field Fs, Fv;
  std::vector<double> hv;
  if (F.dir_freqs > 0) {
    split_nets(F, Fs, Fv);
    rt.e.assign(6 * F.dir_freqs, 0.0);
    direnc(d, F.dir_freqs, rt.e.data());
    hv.assign(F.K + 6 * F.dir_freqs, 0.0);
  }
  double tau_prev = 0.0;
  for (int j = 0; j < S; ++j) {
    double t = nearv + (double)j * rt.delta;
    rt.t[j] = t;
    double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    contract(F, x);
    sample_taps(F, x, rt.taps[j]);
    gather(F, rt.taps[j], h.data());
    if (F.dir_freqs > 0) {   // sigma = g_sigma(h), c = g_v(h, direnc(d))
      mlp_forward(Fs, h.data(), rt.mlp[j]);
      for (int k = 0; k < F.K; ++k) hv[k] = h[k];
      for (size_t k = 0; k < rt.e.size(); ++k) hv[F.K + k] = rt.e[k];
      mlp_forward(Fv, hv.data(), rt.mlpv[j]);
      rt.sigma[j] = softplus(rt.mlp[j].a[F.n_layers][0]);
      for (int k = 0; k < C; ++k) rt.c[j][k] = sigmoid(rt.mlpv[j].a[F.n_layers][k]);
    } else {
      mlp_forward(F, h.data(), rt.mlp[j]);
      const std::vector<double>& out = rt.mlp[j].a[F.n_layers];
      rt.sigma[j] = softplus(out[0]);
      for (int k = 0; k < C; ++k) rt.c[j][k] = sigmoid(out[1 + k]);
    }
    double ds = rt.delta * rt.sigma[j];
    rt.tau[j] = tau_prev + ds;
    rt.T[j] = std::exp(-rt.tau[j]);
    rt.w[j] = (j == 0) ? 0.0 : std::exp(-tau_prev) * (-std::expm1(-ds));
    tau_prev = rt.tau[j];
  }
}

// out = sum_{j>=1} w_j c_j + T_R bg; tau_out = tau_R; depth (optional, reading
// R26: the "depths" feature of P:234 composited like a colour, no background
// term) = sum_{j>=1} w_j t_j.
void finish_forward(const Field& F, const RayTrace& rt, const double* bg, double* out, double* tau_out,
                    double* depth_out) {
  const int C = F.widths[F.n_layers] - 1;
  const int R = rt.S - 1;
  for (int k = 0; k < C; ++k) {
    double v = 0.0;
    for (int j = 1; j <= R; ++j) v += rt.w[j] * rt.c[j][k];
    out[k] = v + rt.T[R] * (bg ? bg[k] : 0.0);
  }
  *tau_out = rt.tau[R];
  if (depth_out) {
    double dep = 0.0;
    for (int j = 1; j <= R; ++j) dep += rt.w[j] * rt.t[j];
    *depth_out = dep;
  }
}

void mlp_slack(const Field& F, const MlpTrace& tr, const double* dout, double band, double* slack_params,
               double* dh_slack);

// O5 / O7: backward for one ray. Loss convention L = p.out + g_tau * tau_R
// (+ g_depth * depth: the depth is one more composited channel whose per-sample
// value t_j has no parameter dependence, so it only enters through a_j).
// mode 0: Eq. 3 via suffix sums over the stored w_j a_j:
//   dL/dsigma_q = -Delta (G_q - [q>=1] T_q a_q) + Delta g_tau,
//   G_q = sum_{j>q} w_j a_j + T_R (p.bg),
//   dL/dc_q = [q>=1] w_q p.
// mode 1: literal derivative of Eq. 1 (O(S^2)):
//   dout/dsigma_q = sum_{j>=1} (dT_{j-1}/dsigma_q - dT_j/dsigma_q) c_j + dT_R/dsigma_q bg,
//   dT_j/dsigma_q = -Delta T_j [q <= j], T_{-1} = 1 (constant).
void backward_ray(const Field& F, const RayTrace& rt, const double* bg, const double* p, double gtau, double gdep,
                  int mode,
                  double* const* grad_planes, double* grad_params, double band = 0.0,
                  double* const* slack_planes = nullptr, double* slack_params = nullptr) {
  const int C = F.widths[F.n_layers] - 1;
  const int S = rt.S, R = S - 1;
  const double Dl = rt.delta;
  std::vector<double> a(S), dsig(S);
  for (int j = 0; j < S; ++j) {
    double s = 0.0;
    for (int k = 0; k < C; ++k) s += p[k] * rt.c[j][k];
    a[j] = s + gdep * rt.t[j];
  }
  double b = 0.0;
  if (bg)
    for (int k = 0; k < C; ++k) b += p[k] * bg[k];
  if (mode == 0) {
    double G = rt.T[R] * b;  // G_R
    for (int q = R; q >= 0; --q) {
      dsig[q] = -Dl * (G - (q >= 1 ? rt.T[q] * a[q] : 0.0)) + Dl * gtau;
      G += rt.w[q] * a[q];     // G_{q-1} = G_q + w_q a_q
    }
  } else {
    for (int q = 0; q < S; ++q) {
      double s = 0.0;
      for (int j = 1; j <= R; ++j) {
        double dTjm1 = (q <= j - 1) ? -Dl * rt.T[j - 1] : 0.0;
        double dTj = (q <= j) ? -Dl * rt.T[j] : 0.0;
        s += (dTjm1 - dTj) * a[j];
      }
      s += -Dl * rt.T[R] * b;  // q <= R always
      dsig[q] = s + Dl * gtau;
    }
  }
  std::vector<double> dout(1 + C), dh(F.K);
  Field Fs, Fv;
  std::vector<double> dhv, dsv;
  int64_t nsig = 0;
  if (F.dir_freqs > 0) {
    split_nets(F, Fs, Fv);
    nsig = net_params(F.n_layers, Fs.widths);
    dhv.assign(F.K + 6 * F.dir_freqs, 0.0);
    dsv.assign(F.K + 6 * F.dir_freqs, 0.0);
  }
  for (int q = 0; q < S; ++q) {
    const double o0 = rt.mlp[q].a[F.n_layers][0];   // density logit (g_sigma's output when split)
    dout[0] = dsig[q] * sigmoid(o0);  // softplus' = sigmoid
    for (int k = 0; k < C; ++k) {
      double dc = (q >= 1) ? rt.w[q] * p[k] : 0.0;
      dout[1 + k] = dc * rt.c[q][k] * (1.0 - rt.c[q][k]);
    }
    if (F.dir_freqs > 0) {   // dL/dh = g_sigma VJP + the h part of the g_v VJP (direnc gets none)
      mlp_backward(Fs, rt.mlp[q], dout.data(), grad_params, dh.data());
      mlp_backward(Fv, rt.mlpv[q], dout.data() + 1, grad_params + nsig, dhv.data());
      for (int k = 0; k < F.K; ++k) dh[k] += dhv[k];
    } else {
      mlp_backward(F, rt.mlp[q], dout.data(), grad_params, dh.data());
    }
    scatter(F, rt.taps[q], dh.data(), grad_planes);
    if (slack_params) {
      std::vector<double> ds(F.K);
      if (F.dir_freqs > 0) {
        mlp_slack(Fs, rt.mlp[q], dout.data(), band, slack_params, ds.data());
        mlp_slack(Fv, rt.mlpv[q], dout.data() + 1, band, slack_params + nsig, dsv.data());
        for (int k = 0; k < F.K; ++k) ds[k] += dsv[k];
      } else {
        mlp_slack(F, rt.mlp[q], dout.data(), band, slack_params, ds.data());
      }
      scatter(F, rt.taps[q], ds.data(), slack_planes);
    }
  }
}

// Slack bound for ambiguous ReLU decisions (test infrastructure for the parity
// metric). For every sample and hidden unit whose
// pre-activation is within band * scale of 0 (scale = sum_k |W_ik a_k| + |b_i|),
// ReLU'(z) may legitimately be evaluated either way by a finite-precision
// implementation. Flipping that one decision changes the unit's delta by
// |s_i| (s = W_{l+1}^T delta_{l+1}, before the mask) and, through the lower
// layers, the parameter and grid gradients. This accumulates an elementwise
// upper bound of |change| (absolute values at every step, masks ignored
// below the flipped unit) into slack buffers with the gradients' shapes.
void mlp_slack(const Field& F, const MlpTrace& tr, const double* dout, double band, double* slack_params,
               double* dh_slack) {
  const int L = F.n_layers;
  std::vector<int64_t> off(L);
  int64_t o = 0;
  for (int l = 0; l < L; ++l) {
    off[l] = o;
    o += (int64_t)F.widths[l + 1] * F.widths[l] + F.widths[l + 1];
  }
  for (int k = 0; k < F.widths[0]; ++k) dh_slack[k] = 0.0;
  // pre-mask upstream s_l for every hidden layer l (the delta of z[l] before ReLU')
  std::vector<std::vector<double>> pre(L);
  std::vector<double> delta(dout, dout + F.widths[L]);
  for (int l = L - 1; l >= 1; --l) {
    int fin = F.widths[l], fout = F.widths[l + 1];
    const double* Wl = F.params + off[l];
    std::vector<double> s(fin, 0.0);
    for (int k = 0; k < fin; ++k)
      for (int i = 0; i < fout; ++i) s[k] += Wl[(int64_t)i * fin + k] * delta[i];
    pre[l - 1] = s;
    for (int k = 0; k < fin; ++k) s[k] = tr.z[l - 1][k] > 0.0 ? s[k] : 0.0;
    delta.swap(s);
  }
  for (int h = 0; h < L - 1; ++h) {
    const int fin = F.widths[h], fout = F.widths[h + 1];
    const double* Wh = F.params + off[h];
    const double* bh = Wh + (int64_t)fout * fin;
    for (int i = 0; i < fout; ++i) {
      double sc = std::fabs(bh[i]);
      for (int k = 0; k < fin; ++k) sc += std::fabs(Wh[(int64_t)i * fin + k] * tr.a[h][k]);
      if (!(std::fabs(tr.z[h][i]) < band * sc)) continue;
      std::vector<double> v(fout, 0.0);
      v[i] = std::fabs(pre[h][i]);
      for (int l = h; l >= 0; --l) {
        const int li = F.widths[l], lo = F.widths[l + 1];
        const double* Wl = F.params + off[l];
        double* sW = slack_params + off[l];
        double* sb = sW + (int64_t)lo * li;
        for (int r = 0; r < lo; ++r) {
          if (v[r] == 0.0) continue;
          sb[r] += v[r];
          for (int k = 0; k < li; ++k) sW[(int64_t)r * li + k] += v[r] * std::fabs(tr.a[l][k]);
        }
        std::vector<double> nv(li, 0.0);
        for (int k = 0; k < li; ++k)
          for (int r = 0; r < lo; ++r) nv[k] += std::fabs(Wl[(int64_t)r * li + k]) * v[r];
        if (l == 0)
          for (int k = 0; k < li; ++k) dh_slack[k] += nv[k];
        v.swap(nv);
      }
    }
  }
}

Field make_field(int kind, int H, int W, int D, int K, const double* p0, const double* p1, const double* p2,
                 int n_layers, const int* widths, const double* params, int contraction = 0,
                 double contract_a = 1.0, int dir_freqs = 0) {
  Field F;
  F.dir_freqs = dir_freqs;
  F.contraction = contraction;
  F.contract_a = contract_a;
  F.kind = kind;
  F.H = H;
  F.W = W;
  F.D = D;
  F.K = K;
  F.plane[0] = p0;
  F.plane[1] = p1;
  F.plane[2] = p2;
  F.n_layers = n_layers;
  F.widths = widths;
  F.params = params;
  return F;
}

int check(int kind, int H, int W, int D, int K, int n_layers, const int* widths, int S) {
  if (kind != 0 && kind != 1) return 1;
  if (H < 2 || W < 2 || D < 2 || K < 1) return 1;
  if (n_layers < 1 || n_layers > 8) return 1;
  if (widths[0] != K || widths[n_layers] < 2) return 1;
  if (S < 2) return 1;
  return 0;
}

}  // namespace

extern "C" {

int lpo_version(void) { return 2; }

// CC(x) for n points (contraction 1 = per-axis, 2 = radial), out[n][3].
int lpo_contract(int contraction, double a, int64_t n, const double* x, double* out) {
  if (contraction < 0 || contraction > 2) return 1;
  Field F = make_field(0, 2, 2, 2, 1, nullptr, nullptr, nullptr, 0, nullptr, nullptr, contraction, a);
  for (int64_t i = 0; i < n; ++i) {
    double p[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    contract(F, p);
    for (int k = 0; k < 3; ++k) out[3 * i + k] = p[k];
  }
  return 0;
}

// h(x) for n points: h_out[n][K].
int lpo_sample(int kind, int H, int W, int D, int K, const double* p0, const double* p1, const double* p2,
               int64_t n, const double* x, double* h_out) {
  int w1[2] = {K, 2};
  if (check(kind, H, W, D, K, 1, w1, 2)) return 1;
  Field F = make_field(kind, H, W, D, K, p0, p1, p2, 0, nullptr, nullptr);
  std::vector<Tap> taps;
  for (int64_t i = 0; i < n; ++i) {
    sample_taps(F, x + 3 * i, taps);
    gather(F, taps, h_out + i * K);
  }
  return 0;
}

// Transpose of lpo_sample: g_planes[c] += sum_i w_{i,c} v_i (accumulates).
int lpo_splat(int kind, int H, int W, int D, int K, int64_t n, const double* x, const double* v, double* g0,
              double* g1, double* g2) {
  int w1[2] = {K, 2};
  if (check(kind, H, W, D, K, 1, w1, 2)) return 1;
  Field F = make_field(kind, H, W, D, K, nullptr, nullptr, nullptr, 0, nullptr, nullptr);
  double* g[3] = {g0, g1, g2};
  std::vector<Tap> taps;
  for (int64_t i = 0; i < n; ++i) {
    sample_taps(F, x + 3 * i, taps);
    scatter(F, taps, v + i * K, g);
  }
  return 0;
}

// MLP forward for n inputs: out[n][widths[n_layers]].
int lpo_mlp_forward(int n_layers, const int* widths, const double* params, int64_t n, const double* in,
                    double* out) {
  Field F = make_field(0, 2, 2, 2, widths[0], nullptr, nullptr, nullptr, n_layers, widths, params);
  MlpTrace tr;
  for (int64_t i = 0; i < n; ++i) {
    mlp_forward(F, in + i * widths[0], tr);
    for (int k = 0; k < widths[n_layers]; ++k) out[i * widths[n_layers] + k] = tr.a[n_layers][k];
  }
  return 0;
}

// MLP VJP for n inputs: accumulates grad_params, writes grad_in[n][K].
int lpo_mlp_backward(int n_layers, const int* widths, const double* params, int64_t n, const double* in,
                     const double* dout, double* grad_params, double* grad_in) {
  Field F = make_field(0, 2, 2, 2, widths[0], nullptr, nullptr, nullptr, n_layers, widths, params);
  MlpTrace tr;
  for (int64_t i = 0; i < n; ++i) {
    mlp_forward(F, in + i * widths[0], tr);
    mlp_backward(F, tr, dout + i * widths[n_layers], grad_params, grad_in + i * widths[0]);
  }
  return 0;
}

// Forward render of rays [r0, r1): out[M][C], tau_out[M] (optical depth tau_R).
int lpo_render_forward(int kind, int H, int W, int D, int K, const double* p0, const double* p1, const double* p2,
                       int n_layers, const int* widths, const double* params, int64_t r0, int64_t r1,
                       const double* origins, const double* dirs, const double* nearv, const double* farv, int S,
                       const double* bg, double* out, double* tau_out, double* depth_out, int contraction,
                       double contract_a, int dir_freqs) {
  if (check(kind, H, W, D, K, n_layers, widths, S)) return 1;
  Field F = make_field(kind, H, W, D, K, p0, p1, p2, n_layers, widths, params, contraction, contract_a,
                       dir_freqs);
  const int C = widths[n_layers] - 1;
  RayTrace rt;
  for (int64_t r = r0; r < r1; ++r) {
    trace_ray(F, origins + 3 * r, dirs + 3 * r, nearv[r], farv[r], S, rt);
    finish_forward(F, rt, bg, out + r * C, tau_out + r, depth_out ? depth_out + r : nullptr);
  }
  return 0;
}

// Backward of rays [r0, r1). grad_* are ACCUMULATED (+=). grad_tau may be NULL.
// mode 0 = Eq. 3 suffix sums, mode 1 = literal O(S^2) derivative.
int lpo_render_backward(int kind, int H, int W, int D, int K, const double* p0, const double* p1, const double* p2,
                        int n_layers, const int* widths, const double* params, int64_t r0, int64_t r1,
                        const double* origins, const double* dirs, const double* nearv, const double* farv, int S,
                        const double* bg, const double* grad_out, const double* grad_tau, double* g0, double* g1,
                        double* g2, double* grad_params, int mode, const double* grad_depth, int contraction,
                        double contract_a, int dir_freqs) {
  if (check(kind, H, W, D, K, n_layers, widths, S)) return 1;
  Field F = make_field(kind, H, W, D, K, p0, p1, p2, n_layers, widths, params, contraction, contract_a,
                       dir_freqs);
  const int C = widths[n_layers] - 1;
  double* g[3] = {g0, g1, g2};
  RayTrace rt;
  for (int64_t r = r0; r < r1; ++r) {
    trace_ray(F, origins + 3 * r, dirs + 3 * r, nearv[r], farv[r], S, rt);
    backward_ray(F, rt, bg, grad_out + r * C, grad_tau ? grad_tau[r] : 0.0, grad_depth ? grad_depth[r] : 0.0, mode,
                 g, grad_params);
  }
  return 0;
}

// Slack bound (see mlp_slack) of rays [r0, r1) accumulated into slack_* with the
// gradient shapes; band = relative |z| below which a ReLU decision is ambiguous.
int lpo_render_relu_slack(int kind, int H, int W, int D, int K, const double* p0, const double* p1,
                          const double* p2, int n_layers, const int* widths, const double* params, int64_t r0,
                          int64_t r1, const double* origins, const double* dirs, const double* nearv,
                          const double* farv, int S, const double* bg, const double* grad_out,
                          const double* grad_tau, double band, double* s0, double* s1, double* s2,
                          double* slack_params, const double* grad_depth, int contraction, double contract_a, int dir_freqs) {
  if (check(kind, H, W, D, K, n_layers, widths, S)) return 1;
  Field F = make_field(kind, H, W, D, K, p0, p1, p2, n_layers, widths, params, contraction, contract_a,
                       dir_freqs);
  const int C = widths[n_layers] - 1;
  double* sg[3] = {s0, s1, s2};
  int64_t np = 0;
  if (dir_freqs > 0) {   // g_sigma then g_v (split_nets)
    Field Fs, Fv;
    split_nets(F, Fs, Fv);
    np = net_params(n_layers, Fs.widths) + net_params(n_layers, Fv.widths);
  } else {
    np = net_params(n_layers, widths);
  }
  std::vector<double> gp(np, 0.0);
  std::vector<std::vector<double>> gg(3);
  double* gptr[3] = {nullptr, nullptr, nullptr};
  const int64_t nel[3] = {(int64_t)H * W * (kind == 1 ? D : 1) * K, (int64_t)W * D * K, (int64_t)D * H * K};
  for (int i = 0; i < (kind == 1 ? 1 : 3); ++i) {
    gg[i].assign(nel[i], 0.0);
    gptr[i] = gg[i].data();
  }
  RayTrace rt;
  for (int64_t r = r0; r < r1; ++r) {
    trace_ray(F, origins + 3 * r, dirs + 3 * r, nearv[r], farv[r], S, rt);
    backward_ray(F, rt, bg, grad_out + r * C, grad_tau ? grad_tau[r] : 0.0, grad_depth ? grad_depth[r] : 0.0, 0,
                 gptr, gp.data(), band, sg, slack_params);
  }
  return 0;
}

// ---------------------------------------------------------------- Splatter
// Each pixel ray i expands into the same R+1 equispaced points as the renderer
// ("R+1 equispaced 3D points", points inheriting the pixel's feature v_i)
// and pushes v_i into theta with the sampling weights of h ("the splatting
// weights are the same as the sampling weights used in rendering"),
// while a second pass pushes the scalar 1 into theta_weight. The
// result is theta / theta_weight, 0 where no weight landed (reading
// R27). The MLP g_s of Eq. 2 is disabled, as in the paper's benchmark.
// Accumulates theta_acc[cells][K] and weight_acc[cells][1] (+=) for rays [r0, r1).
int lpo_splat_rays(int kind, int H, int W, int D, int K, int64_t r0, int64_t r1, const double* origins,
                   const double* dirs, const double* nearv, const double* farv, int S, const double* features,
                   double* t0, double* t1, double* t2, double* w0, double* w1, double* w2, int contraction,
                   double contract_a) {
  int wd[2] = {K, 2};
  if (check(kind, H, W, D, K, 1, wd, S)) return 1;
  Field F = make_field(kind, H, W, D, K, nullptr, nullptr, nullptr, 0, nullptr, nullptr, contraction, contract_a);
  Field F1 = make_field(kind, H, W, D, 1, nullptr, nullptr, nullptr, 0, nullptr, nullptr, contraction, contract_a);
  double* tg[3] = {t0, t1, t2};
  double* wg[3] = {w0, w1, w2};
  const double one = 1.0;
  const int R = S - 1;
  std::vector<Tap> taps;
  for (int64_t r = r0; r < r1; ++r) {
    const double* o = origins + 3 * r;
    const double* d = dirs + 3 * r;
    double span = farv[r] - nearv[r];
    double delta = (span > 0.0 ? span : 0.0) / (double)R;
    for (int j = 0; j < S; ++j) {
      double t = nearv[r] + (double)j * delta;
      double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
      contract(F, x);
      sample_taps(F, x, taps);
      scatter(F, taps, features + r * K, tg);     // pass 1: the pixel feature
      scatter(F1, taps, &one, wg);                // pass 2: the scalar 1 (MLPs off)
    }
  }
  return 0;
}

// theta / theta_weight per cell (0 where theta_weight == 0), n cells of K channels.
int lpo_splat_normalize(int64_t n, int K, const double* theta, const double* weight, double* out) {
  for (int64_t c = 0; c < n; ++c)
    for (int k = 0; k < K; ++k) out[c * K + k] = weight[c] > 0.0 ? theta[c * K + k] / weight[c] : 0.0;
  return 0;
}

// Backward of the normalised splat w.r.t. the features of rays [r0, r1):
// theta_weight is geometry only and treated as a constant ("manually cache
// theta_weight to normalize gradients"), so with g' = grad_out / theta_weight
// (0 where theta_weight == 0), dL/dv_i = sum_j h_{g'}(x_ij), the renderer's
// gather ("mirrors"). grad_features[M][K] is overwritten for those rays.
int lpo_splat_rays_backward(int kind, int H, int W, int D, int K, int64_t r0, int64_t r1, const double* origins,
                            const double* dirs, const double* nearv, const double* farv, int S, const double* g0,
                            const double* g1, const double* g2, const double* w0, const double* w1,
                            const double* w2, double* grad_features, int contraction, double contract_a) {
  int wd[2] = {K, 2};
  if (check(kind, H, W, D, K, 1, wd, S)) return 1;
  Field F = make_field(kind, H, W, D, K, nullptr, nullptr, nullptr, 0, nullptr, nullptr, contraction, contract_a);
  const double* gg[3] = {g0, g1, g2};
  const double* wg[3] = {w0, w1, w2};
  const int R = S - 1;
  std::vector<Tap> taps;
  for (int64_t r = r0; r < r1; ++r) {
    const double* o = origins + 3 * r;
    const double* d = dirs + 3 * r;
    double span = farv[r] - nearv[r];
    double delta = (span > 0.0 ? span : 0.0) / (double)R;
    double* gv = grad_features + r * K;
    for (int k = 0; k < K; ++k) gv[k] = 0.0;
    for (int j = 0; j < S; ++j) {
      double t = nearv[r] + (double)j * delta;
      double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
      contract(F, x);
      sample_taps(F, x, taps);
      for (const Tap& tp : taps) {
        double wc = wg[tp.plane][tp.cell];
        if (!(wc > 0.0)) continue;
        const double* g = gg[tp.plane] + tp.cell * K;
        for (int k = 0; k < K; ++k) gv[k] += tp.w * (g[k] / wc);
      }
    }
  }
  return 0;
}

// ---------------------------------------------------------------- Splatter with g_s (Eq. 2)
// v~_ij = g_s(v_i, h_prior(x_ij), direnc(d_i)) (reading R30): the input is the
// concatenation [v_i (C_in) ; h_prior(x_ij) (K_p, the prior grid theta^ sampled
// with the same scheme h, same kind and dims as theta) ; direnc(d_i) (6F)], g_s
// an MLP (ReLU hidden, identity output) with widths[0] = C_in + K_p + 6F and
// widths[L] = K (theta's channels). Pass 1 splats v~_ij, pass 2 (MLPs off,
// P:748) splats 1 into theta_weight exactly as lpo_splat_rays.
struct SplatMlp {
  Field F;        // target geometry (K = C_out), contraction
  Field Fp;       // prior grid (K = K_p)
  Field Fm;       // g_s (widths / params)
  int C_in, F_dir;
};

SplatMlp make_splat_mlp(int kind, int H, int W, int D, int K, int Kp, const double* q0, const double* q1,
                        const double* q2, int n_layers, const int* widths, const double* params, int C_in, int F_dir,
                        int contraction, double contract_a) {
  SplatMlp m;
  m.F = make_field(kind, H, W, D, K, nullptr, nullptr, nullptr, 0, nullptr, nullptr, contraction, contract_a);
  m.Fp = make_field(kind, H, W, D, Kp, q0, q1, q2, 0, nullptr, nullptr, contraction, contract_a);
  m.Fm = make_field(kind, H, W, D, widths[0], nullptr, nullptr, nullptr, n_layers, widths, params);
  m.C_in = C_in;
  m.F_dir = F_dir;
  return m;
}

// u = [v ; h_prior(x) ; direnc(d)] and the prior taps of point x
void splat_mlp_input(const SplatMlp& m, const double* v, const double* x, const double* e, std::vector<Tap>& taps,
                     std::vector<double>& u) {
  const int Kp = m.Fp.K;
  u.assign(m.Fm.widths[0], 0.0);
  for (int k = 0; k < m.C_in; ++k) u[k] = v[k];
  sample_taps(m.Fp, x, taps);
  gather(m.Fp, taps, u.data() + m.C_in);
  for (int k = 0; k < 6 * m.F_dir; ++k) u[m.C_in + Kp + k] = e[k];
}

int lpo_splat_rays_mlp(int kind, int H, int W, int D, int K, int Kp, const double* q0, const double* q1,
                       const double* q2, int n_layers, const int* widths, const double* params, int C_in, int F_dir,
                       int64_t r0, int64_t r1, const double* origins, const double* dirs, const double* nearv,
                       const double* farv, int S, const double* features, double* t0, double* t1, double* t2,
                       double* w0, double* w1, double* w2, int contraction, double contract_a) {
  if (widths[0] != C_in + Kp + 6 * F_dir || widths[n_layers] != K || S < 2) return 1;
  SplatMlp m = make_splat_mlp(kind, H, W, D, K, Kp, q0, q1, q2, n_layers, widths, params, C_in, F_dir, contraction,
                              contract_a);
  Field F1 = make_field(kind, H, W, D, 1, nullptr, nullptr, nullptr, 0, nullptr, nullptr, contraction, contract_a);
  double* tg[3] = {t0, t1, t2};
  double* wg[3] = {w0, w1, w2};
  const double one = 1.0;
  const int R = S - 1;
  std::vector<Tap> taps, ptaps;
  std::vector<double> u, e(6 * F_dir);
  MlpTrace tr;
  for (int64_t r = r0; r < r1; ++r) {
    const double* o = origins + 3 * r;
    const double* d = dirs + 3 * r;
    direnc(d, F_dir, e.data());
    double span = farv[r] - nearv[r];
    double delta = (span > 0.0 ? span : 0.0) / (double)R;
    for (int j = 0; j < S; ++j) {
      double t = nearv[r] + (double)j * delta;
      double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
      contract(m.F, x);
      sample_taps(m.F, x, taps);
      if (taps.empty()) continue;                 // nothing to splat outside the cube
      splat_mlp_input(m, features + r * C_in, x, e.data(), ptaps, u);
      mlp_forward(m.Fm, u.data(), tr);
      scatter(m.F, taps, tr.a[n_layers].data(), tg);   // pass 1: v~_ij
      scatter(F1, taps, &one, wg);                     // pass 2: 1 (MLPs off)
    }
  }
  return 0;
}

// Backward of the normalised g_s splat (theta_weight constant): per sample
// dv~_ij = h_{g'}(x_ij), g' = grad_out / theta_weight; then the g_s VJP gives
// dL/dv_i (summed over j, overwritten for rays [r0, r1)), the prior gradient
// (scattered with the prior's sampling weights, accumulated) and the g_s
// parameter gradient (accumulated).
int lpo_splat_rays_mlp_backward(int kind, int H, int W, int D, int K, int Kp, const double* q0, const double* q1,
                                const double* q2, int n_layers, const int* widths, const double* params, int C_in,
                                int F_dir, int64_t r0, int64_t r1, const double* origins, const double* dirs,
                                const double* nearv, const double* farv, int S, const double* features,
                                const double* g0, const double* g1, const double* g2, const double* w0,
                                const double* w1, const double* w2, double* grad_features, double* gp0, double* gp1,
                                double* gp2, double* grad_params, int contraction, double contract_a) {
  if (widths[0] != C_in + Kp + 6 * F_dir || widths[n_layers] != K || S < 2) return 1;
  SplatMlp m = make_splat_mlp(kind, H, W, D, K, Kp, q0, q1, q2, n_layers, widths, params, C_in, F_dir, contraction,
                              contract_a);
  const double* gg[3] = {g0, g1, g2};
  const double* wg[3] = {w0, w1, w2};
  double* gpr[3] = {gp0, gp1, gp2};
  const int R = S - 1;
  std::vector<Tap> taps, ptaps;
  std::vector<double> u, e(6 * F_dir), dv(K), du(widths[0]);
  MlpTrace tr;
  for (int64_t r = r0; r < r1; ++r) {
    const double* o = origins + 3 * r;
    const double* d = dirs + 3 * r;
    direnc(d, F_dir, e.data());
    double span = farv[r] - nearv[r];
    double delta = (span > 0.0 ? span : 0.0) / (double)R;
    double* gv = grad_features + r * C_in;
    for (int k = 0; k < C_in; ++k) gv[k] = 0.0;
    for (int j = 0; j < S; ++j) {
      double t = nearv[r] + (double)j * delta;
      double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
      contract(m.F, x);
      sample_taps(m.F, x, taps);
      if (taps.empty()) continue;
      for (int k = 0; k < K; ++k) dv[k] = 0.0;
      for (const Tap& tp : taps) {
        double wc = wg[tp.plane][tp.cell];
        if (!(wc > 0.0)) continue;
        const double* g = gg[tp.plane] + tp.cell * K;
        for (int k = 0; k < K; ++k) dv[k] += tp.w * (g[k] / wc);
      }
      splat_mlp_input(m, features + r * C_in, x, e.data(), ptaps, u);
      mlp_forward(m.Fm, u.data(), tr);
      mlp_backward(m.Fm, tr, dv.data(), grad_params, du.data());
      for (int k = 0; k < C_in; ++k) gv[k] += du[k];
      scatter(m.Fp, ptaps, du.data() + C_in, gpr);   // prior gradient
    }
  }
  return 0;
}

// Slack bound for ambiguous ReLU decisions of g_s (the parity metric's
// allowance, as lpo_render_relu_slack for the renderer; DESIGN.md "Parity
// metric"): for every in-cube sample and g_s hidden unit with |z| < band *
// (sum_k |W_ik u_k| + |b_i|), mlp_slack bounds the change of the g_s parameter
// gradient and of dL/du when the decision flips; the u-part splits into the
// feature slack of the ray (first C_in entries, accumulated over its samples)
// and the prior slack (next K_p entries, pushed with the prior's sampling
// weights, which are >= 0). Accumulates (+=) into slack_features[M][C_in],
// slack_prior planes and slack_params.
int lpo_splat_mlp_relu_slack(int kind, int H, int W, int D, int K, int Kp, const double* q0, const double* q1,
                             const double* q2, int n_layers, const int* widths, const double* params, int C_in,
                             int F_dir, int64_t r0, int64_t r1, const double* origins, const double* dirs,
                             const double* nearv, const double* farv, int S, const double* features,
                             const double* g0, const double* g1, const double* g2, const double* w0,
                             const double* w1, const double* w2, double band, double* slack_features, double* sp0,
                             double* sp1, double* sp2, double* slack_params, int contraction, double contract_a) {
  if (widths[0] != C_in + Kp + 6 * F_dir || widths[n_layers] != K || S < 2) return 1;
  SplatMlp m = make_splat_mlp(kind, H, W, D, K, Kp, q0, q1, q2, n_layers, widths, params, C_in, F_dir, contraction,
                              contract_a);
  const double* gg[3] = {g0, g1, g2};
  const double* wg[3] = {w0, w1, w2};
  double* spr[3] = {sp0, sp1, sp2};
  const int R = S - 1;
  std::vector<Tap> taps, ptaps;
  std::vector<double> u, e(6 * F_dir), dv(K), du_slack(widths[0]);
  MlpTrace tr;
  for (int64_t r = r0; r < r1; ++r) {
    const double* o = origins + 3 * r;
    const double* d = dirs + 3 * r;
    direnc(d, F_dir, e.data());
    double span = farv[r] - nearv[r];
    double delta = (span > 0.0 ? span : 0.0) / (double)R;
    for (int j = 0; j < S; ++j) {
      double t = nearv[r] + (double)j * delta;
      double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
      contract(m.F, x);
      sample_taps(m.F, x, taps);
      if (taps.empty()) continue;
      for (int k = 0; k < K; ++k) dv[k] = 0.0;
      for (const Tap& tp : taps) {
        double wc = wg[tp.plane][tp.cell];
        if (!(wc > 0.0)) continue;
        const double* g = gg[tp.plane] + tp.cell * K;
        for (int k = 0; k < K; ++k) dv[k] += tp.w * (g[k] / wc);
      }
      splat_mlp_input(m, features + r * C_in, x, e.data(), ptaps, u);
      mlp_forward(m.Fm, u.data(), tr);
      mlp_slack(m.Fm, tr, dv.data(), band, slack_params, du_slack.data());
      for (int k = 0; k < C_in; ++k) slack_features[r * C_in + k] += du_slack[k];
      scatter(m.Fp, ptaps, du_slack.data() + C_in, spr);
    }
  }
  return 0;
}

// Per-sample trace of one ray for invariant tests: sigma[S], tau[S], T[S], w[S], c[S][C].
int lpo_trace(int kind, int H, int W, int D, int K, const double* p0, const double* p1, const double* p2,
              int n_layers, const int* widths, const double* params, const double* origin, const double* dir,
              double nearv, double farv, int S, double* sigma, double* tau, double* T, double* w, double* c,
              int contraction, double contract_a, int dir_freqs) {
  if (check(kind, H, W, D, K, n_layers, widths, S)) return 1;
  Field F = make_field(kind, H, W, D, K, p0, p1, p2, n_layers, widths, params, contraction, contract_a,
                       dir_freqs);
  const int C = widths[n_layers] - 1;
  RayTrace rt;
  trace_ray(F, origin, dir, nearv, farv, S, rt);
  for (int j = 0; j < S; ++j) {
    sigma[j] = rt.sigma[j];
    tau[j] = rt.tau[j];
    T[j] = rt.T[j];
    w[j] = rt.w[j];
    for (int k = 0; k < C; ++k) c[j * C + k] = rt.c[j][k];
  }
  return 0;
}

}  // extern "C"
