// synth.cuh -- argument block of the Fourier/Mueller synthesis kernel.
#pragma once

#include "kernels.cuh"

namespace vrte {

struct SynthArgs {
    int N, L, n_in, n_dphi;
    const double* up;           // [slot][4 n_in][4N] tau=0 upward stacks
    const int* slot_of_order;   // [L] -> slot in `up`
    const double* trig;         // [L][n_dphi][2] cos(m x), sin(m x), x = -dphi
    const double* post;         // [n_in][16] row-major T_ii
    double* out;                // [n_in][N - out_lo][n_dphi][16]
    DeviceStatus* status;
    const double* pre;          // [N][16] row-major left factor per output node (null: identity)
    int out_lo;                 // first output node (Fresnel interface: the refraction cone)
};

void launch_synth(const SynthArgs& a, cudaStream_t st);

}  // namespace vrte
