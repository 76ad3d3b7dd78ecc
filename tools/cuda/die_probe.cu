// die_probe.cu -- which of the B200's two dies each SM sits on (experiment tool).
// Each SM times dependent L2 hits (ld.global.cg) on NL lines 2 KB apart; a line homed on the
// SM's own die answers ~28 cycles faster (B300_MICROARCH.md "SM->L2-die routing").  Per line
// the SMs split into a fast and a slow group; the split is the die map up to a flip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/die_probe tools/cuda/die_probe.cu
#include <cstdio>
#include <vector>
#include <algorithm>
__global__ void probe(const unsigned* buf, int nl, int reps, unsigned long long* out) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x != 0) return;
  unsigned v = 0;
  for (int l = 0; l < nl; ++l) {
    const unsigned* a = buf + (size_t)l * 512;   // 2 KB apart
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(a + v));
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(a + v));
    const long long t1 = clock64();
    out[(size_t)blockIdx.x * nl + l] = (unsigned long long)(t1 - t0) | ((unsigned long long)smid << 48);
  }
  if (v == 12345) out[0] = 0;
}
int main() {
  const int nl = 64, reps = 64, nb = 148 * 2;
  unsigned* buf; unsigned long long* out;
  cudaMalloc(&buf, (size_t)nl * 2048);
  cudaMemset(buf, 0, (size_t)nl * 2048);
  cudaMalloc(&out, (size_t)nb * nl * 8);
  probe<<<nb, 32>>>(buf, nl, reps, out);
  probe<<<nb, 32>>>(buf, nl, reps, out);
  std::vector<unsigned long long> h((size_t)nb * nl);
  cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<std::vector<double>> lat(148, std::vector<double>(nl, 0.0));
  std::vector<int> cnt(148, 0);
  for (int b = 0; b < nb; ++b) {
    const int sm = (int)(h[(size_t)b * nl] >> 48);
    cnt[sm]++;
    for (int l = 0; l < nl; ++l)
      lat[sm][l] += (double)(h[(size_t)b * nl + l] & 0xFFFFFFFFFFFFull) / reps;
  }
  // per line: fast/slow split at the midpoint of min and max; align lines to line 0
  std::vector<int> votes(148, 0);
  std::vector<int> ref;
  for (int l = 0; l < nl; ++l) {
    double lo = 1e30, hi = 0;
    for (int s = 0; s < 148; ++s) if (cnt[s]) { double x = lat[s][l] / cnt[s]; lo = std::min(lo, x); hi = std::max(hi, x); }
    const double mid = 0.5 * (lo + hi);
    std::vector<int> g(148, 0);
    for (int s = 0; s < 148; ++s) if (cnt[s]) g[s] = lat[s][l] / cnt[s] < mid;
    if (ref.empty()) ref = g;
    int agree = 0;
    for (int s = 0; s < 148; ++s) agree += g[s] == ref[s];
    const bool flip = agree < 74;
    for (int s = 0; s < 148; ++s) votes[s] += (g[s] ^ flip) ? 1 : -1;
    if (l < 4) printf("line %d: fast %.1f slow %.1f cycles/load\n", l, lo, hi);
  }
  int n0 = 0;
  printf("die map (smid: die):\n");
  for (int s = 0; s < 148; ++s) { const int d = votes[s] > 0; n0 += d == 0; printf("%d%s", d, (s % 37 == 36) ? "\n" : ""); }
  printf("\ndie0 %d SMs, die1 %d SMs; min |vote| = %d of %d\n", n0, 148 - n0,
         abs(*std::min_element(votes.begin(), votes.end(), [](int a, int b) { return abs(a) < abs(b); })), nl);
  return 0;
}
