// tests/native/core_host_capi.cpp -- TEST-ONLY host instantiation of the
// device core (paper_2507_21686_b200/csrc/sphbi_core.cuh), used by the CPU
// test tier to check the core's math against the oracle without a GPU. The
// product path never loads this library: it runs the same header as sm_100a
// code inside libsphbi_cuda.so.
#include <cstdint>
#include <thread>
#include <vector>

#include "../../paper_2507_21686_b200/csrc/sphbi_core.cuh"

using namespace sphbi_dev;

extern "C" {

int core_host_eval_pair(const double* coef, int ncoef, double c2, double qx, double qy, double h,
                        const double* tri6, const double* vals3, int mode, double* out,
                        unsigned long long* counters, int* n_regions) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  return (int)eval_pair(K, qx, qy, h, tri6, vals3, mode, out, counters, n_regions);
}

int core_host_eval_pairs(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                         const double* tri6, const double* vals3, const double* coef, int ncoef,
                         double c2, double h, int nthreads, double* out4, unsigned* status) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int tid) {
    for (int64_t k = tid; k < npairs; k += nthreads) {
      const int64_t i = pp ? pp[k] : k;
      const int64_t t = pt ? pt[k] : k;
      status[k] = eval_pair(K, pxy[2 * i], pxy[2 * i + 1], h, tri6 + 6 * t, vals3 + 3 * t, 0,
                            out4 + 4 * k, nullptr, nullptr);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return 0;
}

double core_host_glibc_hypot(double x, double y) { return glibc_hypot(x, y); }

}  // extern "C"
