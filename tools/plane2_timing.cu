// plane2_timing.cu - where a K = 1 cost call's plane2_kernel time goes, per CTA, from %globaltimer
// stamps (plane2.cuh, built with -DDVQLS_PLANE2_TS): entry, after pdl_wait, x staged, last task
// done (per pair and per CTA), piece reduction written, CTA end.  cfg3 shape (n = 10, d = 10,
// L = 64 random Pauli strings, uniform b), dvqls_cost_dev with K = 1 on the production path
// (CUDA graph, PDL behind the prefix).  Prints min / median / max over the 148 CTAs of each stamp,
// in microseconds after the earliest CTA's pdl_wait return.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDVQLS_PLANE2_TS -diag-suppress 177,550 \
//        -I paper_2604_14435_b200/csrc tools/plane2_timing.cu paper_2604_14435_b200/csrc/*.cu -ldl -o tools/plane2_timing
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "../include/dvqls.h"
namespace dvqls { void* plane2_ts_ptr(); }

int main(int argc, char** argv) {
  const int n = 10, d = 10, L = 64, P = 3 * n * d, K = argc > 1 ? atoi(argv[1]) : 1;
  std::mt19937 rng(7);
  std::set<std::string> seen;
  std::string chars;
  while ((int)seen.size() < L) {
    std::string s;
    for (int q = 0; q < n; ++q) s += "IXYZ"[rng() % 4];
    if (seen.insert(s).second) chars += s;
  }
  std::vector<double> co(2 * L), th(size_t(P) * K);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (auto& c : co) c = u(rng);
  for (auto& t : th) t = 3.0 * u(rng);
  dvqls_bprep b{DVQLS_B_UNIFORM, nullptr};
  dvqls_ctx* ctx = nullptr;
  int rc = dvqls_create(&ctx, n, d, L, chars.data(), co.data(), &b, nullptr);
  if (rc) { printf("create failed %d\n", rc); return 1; }
  double *dth, *dout;
  cudaMalloc(&dth, sizeof(double) * th.size());
  cudaMalloc(&dout, sizeof(double) * 5 * K);
  cudaMemcpy(dth, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice);
  for (int i = 0; i < 30; ++i) rc |= dvqls_cost_dev(ctx, K, dth, dout);
  cudaDeviceSynchronize();
  if (rc) { printf("cost failed %d: %s\n", rc, dvqls_last_error(ctx)); return 1; }
  std::vector<unsigned long long> ts(160 * 16);
  cudaMemcpy(ts.data(), dvqls::plane2_ts_ptr(), sizeof(unsigned long long) * ts.size(), cudaMemcpyDeviceToHost);
  const int G = 148;
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < G; ++c) t0 = std::min(t0, ts[c * 16 + 1]);
  const char* names[12] = {"entry", "pdl_wait", "x_staged", "tasks_done", "reduced", "cta_end",
                           "pair0", "pair1", "pair2", "pair3", "pair4", "pair5"};
  printf("{\"K\": %d, \"note\": \"us after the earliest pdl_wait return; min / median / max over %d CTAs\"", K, G);
  for (int k = 0; k < 12; ++k) {
    std::vector<double> v;
    for (int c = 0; c < G; ++c) v.push_back((double(ts[c * 16 + k]) - double(t0)) * 1e-3);
    std::sort(v.begin(), v.end());
    printf(", \"%s\": [%.2f, %.2f, %.2f]", names[k], v.front(), v[G / 2], v.back());
  }
  // per-CTA spread of its pairs' finish times
  std::vector<double> spread;
  for (int c = 0; c < G; ++c) {
    double lo = 1e30, hi = -1e30;
    for (int p = 0; p < 6; ++p) { double x = double(ts[c * 16 + 6 + p]); lo = std::min(lo, x); hi = std::max(hi, x); }
    spread.push_back((hi - lo) * 1e-3);
  }
  std::sort(spread.begin(), spread.end());
  printf(", \"pair_spread_in_cta\": [%.2f, %.2f, %.2f]}\n", spread.front(), spread[G / 2], spread.back());
  dvqls_destroy(ctx);
  return 0;
}
