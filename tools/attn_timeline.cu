// Per-CTA timeline of the dK/dV backward kernel at the C2 shape (B 8, S 2048, H 28, hd 128):
// the kernel source compiled with HLM_ATTN_TIMELINE, which stamps %globaltimer at CTA start,
// K/V landed (MMA warp), first S/dP landed, last P/dS handed over, accumulators done and CTA
// end. Prints a summary (prologue, per-step time, epilogue, gaps between CTAs on one SM).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -DHLM_ATTN_TIMELINE \
//     -I include -I paper_2602_04816_b200/csrc/kernels tools/attn_timeline.cu -o tools/attn_timeline
#include "../paper_2602_04816_b200/csrc/kernels/attention_tc.cu"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

void hlm_count_launches(long long) {}

int main() {
  const int B = 8, S = 2048, H = 28, ld = H * HD;
  const size_t T = (size_t)B * S, elems = T * ld;
  std::vector<__nv_bfloat16> hbuf(elems);
  unsigned x = 12345;
  for (auto& v : hbuf) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16(((x >> 8) * (1.0f / 16777216.0f) - 0.5f) * 2.0f);
  }
  void *q, *k, *v, *dout, *dq, *dk, *dv;
  float *lse, *dsum;
  for (void** p : {&q, &k, &v, &dout, &dq, &dk, &dv}) {
    cudaMalloc(p, elems * 2);
    cudaMemcpy(*p, hbuf.data(), elems * 2, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&lse, (size_t)B * H * S * 4);
  cudaMalloc(&dsum, (size_t)B * H * S * 4);
  cudaMemset(lse, 0, (size_t)B * H * S * 4);
  cudaMemset(dsum, 0, (size_t)B * H * S * 4);
  const int ctas = (S / TQ) * B * H;
  unsigned long long* tl;
  cudaMalloc(&tl, (size_t)2 * ctas * 16 * 8);
  cudaMemcpyToSymbol(g_attn_tl, &tl, sizeof(tl));
  if (std::getenv("TIMELINE_FWD")) {
    setenv("HLM_ATTN_FWD_PERSIST", "0", 1);   // the stamps are in the one-CTA-per-pair kernel   // flash_fwd_pp2: 0 start, 1 Q landed, 2 tile B's first S,
                                       // 3 tile B's O final, 4 tile B's O stored, 5 end, 6 SM, 7 steps
    const int fctas = (S / 256) * B * H;
    for (int rep = 0; rep < 3; ++rep)
      if (hlm_flash_fwd_tc(q, k, v, dq, lse, B, S, H, ld, 0) != 0) return 1;
    if (cudaDeviceSynchronize() != cudaSuccess) return 2;
    std::vector<unsigned long long> f((size_t)fctas * 16);
    cudaMemcpy(f.data(), tl, f.size() * 8, cudaMemcpyDeviceToHost);
    double q = 0, s0 = 0, fin = 0, st = 0, end = 0, gap = 0;
    int ngap = 0;
    std::map<int, std::vector<std::pair<unsigned long long, unsigned long long>>> per_sm;
    std::map<int, std::vector<double>> by_n;
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int c = 0; c < fctas; ++c) {
      const unsigned long long* r = &f[c * 16];
      t0 = std::min(t0, r[0]);
      t1 = std::max(t1, r[5]);
      q += double(r[1] - r[0]);
      s0 += double(r[2] - r[0]);
      fin += double(r[3] - r[0]);
      st += double(r[4] - r[3]);
      end += double(r[5] - r[4]);
      per_sm[(int)r[6]].push_back({r[0], r[5]});
      by_n[(int)r[7]].push_back(double(r[5] - r[0]));
    }
    for (auto& [sm, v] : per_sm) {
      std::sort(v.begin(), v.end());
      for (size_t i = 1; i < v.size(); ++i) {
        gap += double(v[i].first) - double(v[i - 1].second);
        ++ngap;
      }
    }
    std::printf("forward span %.1f us, %d CTAs; per CTA (us): start -> Q landed %.2f, -> first S %.2f, "
                "-> O final %.2f, O store %.2f, -> end %.2f; gap between CTAs on an SM %.2f\n",
                (t1 - t0) / 1e3, fctas, q / fctas / 1e3, s0 / fctas / 1e3, fin / fctas / 1e3, st / fctas / 1e3,
                end / fctas / 1e3, gap / ngap / 1e3);
    for (auto& [n, v] : by_n) {
      double sum = 0;
      for (double d : v) sum += d;
      std::printf("  %2d key steps: %4zu CTAs, avg %.2f us\n", n, v.size(), sum / v.size() / 1e3);
    }
    return 0;
  }
  for (int rep = 0; rep < 3; ++rep)
    if (hlm_flash_bwd_tc(q, k, v, dout, lse, dsum, dq, dk, dv, B, S, H, ld, 0) != 0) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  std::vector<unsigned long long> h16((size_t)ctas * 16), h((size_t)ctas * 8);
  cudaMemcpy(h16.data(), tl + (std::getenv("TIMELINE_DQ") ? (size_t)ctas * 16 : 0), h16.size() * 8,
             cudaMemcpyDeviceToHost);
  for (int c = 0; c < ctas; ++c)
    for (int k = 0; k < 8; ++k) h[c * 8 + k] = h16[c * 16 + k];

  const bool persist = std::getenv("HLM_ATTN_BWD_PERSIST") == nullptr || std::atoi(std::getenv("HLM_ATTN_BWD_PERSIST"));
  // flash_bwd_dq_tc3 stamps the records after dK/dV's (TIMELINE_DQ=1 analyses those)
  const bool dq_kernel = std::getenv("TIMELINE_DQ") != nullptr;
  if (persist) {
    // records per tile: 0 fetched, 1 first S/dP landed, 2 last P/dS handed over, 3 accumulators
    // done, 4 dK/dV stored (elementwise warp 4), 6 SM, 7 steps
    double fetch_to_s = 0, step = 0, tail = 0, epi = 0, between = 0;
    int nstep = 0, nb = 0;
    std::map<int, std::vector<std::pair<unsigned long long, unsigned long long>>> per_sm;
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int c = 0; c < ctas; ++c) {
      const unsigned long long* r = &h[c * 8];
      const int n = (int)r[7];
      t0 = std::min(t0, r[0]);
      t1 = std::max(t1, r[4]);
      fetch_to_s += double(r[1] - r[0]);
      if (n > 1) {
        step += double(r[2] - r[1]) / (n - 1);
        ++nstep;
      }
      tail += double(r[3] - r[2]);
      epi += double(r[4] - r[3]);
      per_sm[(int)r[6]].push_back({r[0], r[4]});
    }
    for (auto& [sm, v] : per_sm) {
      std::sort(v.begin(), v.end());
      for (size_t i = 1; i < v.size(); ++i) {
        between += double(v[i].first) - double(v[i - 1].second);
        ++nb;
      }
    }
    std::printf(dq_kernel ? "persistent dQ: span %.1f us, %d tiles on %zu SMs\n" : "persistent dK/dV: span %.1f us, %d tiles on %zu SMs\n", (t1 - t0) / 1e3, ctas, per_sm.size());
    std::printf("per tile (us): fetched -> first S/dP landed %.2f, steady step %.3f, last P/dS -> accumulators "
                "%.2f, store %.2f; previous tile stored -> next fetched %.2f\n",
                fetch_to_s / ctas / 1e3, step / nstep / 1e3, tail / ctas / 1e3, epi / ctas / 1e3,
                between / nb / 1e3);
    if (dq_kernel) {   // slot 5: the next tile's Q / dO written to TMEM (before the dQ accumulator wait)
      double nextq = 0, accw = 0;
      for (int c = 0; c < ctas; ++c) {
        const unsigned long long* r = &h[c * 8];
        nextq += double(r[5] - r[2]);
        accw += double(r[3] - r[5]);
      }
      std::printf("dQ boundary (us): last dS -> next tile's Q/dO in TMEM %.2f, then -> dQ accumulator %.2f\n",
                  nextq / ctas / 1e3, accw / ctas / 1e3);

    }
    return 0;
  }
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int c = 0; c < ctas; ++c) {
    t0 = std::min(t0, h[c * 8 + 0]);
    t1 = std::max(t1, h[c * 8 + 5]);
  }
  double pro = 0, kv = 0, step = 0, epi = 0, dur = 0, tail_acc = 0;
  int nstep_cta = 0;
  std::map<int, std::vector<std::pair<unsigned long long, unsigned long long>>> per_sm;
  std::map<int, std::vector<double>> by_n;
  for (int c = 0; c < ctas; ++c) {
    const unsigned long long* r = &h[c * 8];
    const int n = (int)r[7];
    kv += (r[1] - r[0]);
    pro += (r[2] - r[0]);
    if (n > 1) {
      step += double(r[3] - r[2]) / (n - 1);
      ++nstep_cta;
    }
    tail_acc += (r[4] - r[3]);
    epi += (r[5] - r[4]);
    dur += (r[5] - r[0]);
    per_sm[(int)r[6]].push_back({r[0], r[5]});
    by_n[n].push_back(double(r[5] - r[0]));
  }
  double gap = 0;
  int ngap = 0;
  for (auto& [sm, v] : per_sm) {
    std::sort(v.begin(), v.end());
    for (size_t i = 1; i < v.size(); ++i) {
      gap += double(v[i].first) - double(v[i - 1].second);
      ++ngap;
    }
  }
  std::printf("dK/dV kernel span %.1f us, %d CTAs on %zu SMs\n", (t1 - t0) / 1e3, ctas, per_sm.size());
  std::printf("per CTA (us): start->K/V landed %.2f, start->first S/dP landed %.2f, steady step %.3f,\n"
              "  last P/dS -> accumulators done %.2f, accumulators -> end (store dK/dV) %.2f, total %.2f\n",
              kv / ctas / 1e3, pro / ctas / 1e3, step / nstep_cta / 1e3, tail_acc / ctas / 1e3, epi / ctas / 1e3,
              dur / ctas / 1e3);
  std::printf("gap between consecutive CTAs on one SM: %.2f us (avg over %d)\n", gap / ngap / 1e3, ngap);
  for (auto& [n, v] : by_n) {
    double s = 0;
    for (double d : v) s += d;
    std::printf("  n=%2d steps: %5zu CTAs, avg %.2f us\n", n, v.size(), s / v.size() / 1e3);
  }
  return 0;
}
