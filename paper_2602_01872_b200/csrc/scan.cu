// scan.cu -- the single-block middle pass of the device-wide scan in scan.cuh.
#include "scan.cuh"

namespace grappa {

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(int64_t* part, int64_t nb) {
    const int64_t per = ceil_div(nb, kScanThreads);
    const int64_t t0 = (int64_t)threadIdx.x * per;
    const int64_t t1 = t0 + per < nb ? t0 + per : nb;
    int64_t s = 0;
    for (int64_t i = t0; i < t1; i++) s += part[i];
    int64_t tot;
    int64_t run = block_exclusive_scan(s, &tot);
    for (int64_t i = t0; i < t1; i++) {
        int64_t v = part[i];
        part[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) part[nb] = tot;
}

}  // namespace grappa
