// Host-side check of the draft-attention work split (vc_kernels.h): every
// task maps back to the warp whose range holds it (the draft kernel and the
// combine derive the same partial slots), ranges tile [0, T), and every
// range holds >= min_tasks tasks.
#include <cstdio>
#include <initializer_list>

#include "vc_kernels.h"

using namespace vc;

int main() {
  long bad = 0, checks = 0;
  {
    for (int nwmax : {2368, 1776, 1000, 64, 1}) {
      for (int T : {1, 7, 100, 1000, 4096, 32768, 131072, 2367, 2369}) {
        for (int mt : {4, 9}) {
          const int nw = draft_active_warps(T, nwmax, mt);
          int minr = 1 << 30;
          for (int w = 0; w < nw; ++w) {
            const int b0 = draft_task_begin(w, T, nw), b1 = draft_task_begin(w + 1, T, nw);
            if (b1 - b0 < minr) minr = b1 - b0;
            for (int t = b0; t < b1; ++t, ++checks)
              if (draft_task_warp(t, T, nw) != w) ++bad;
          }
          if (draft_task_begin(0, T, nw) != 0 || draft_task_begin(nw, T, nw) != T) ++bad;
          if (T >= mt && nw > 1 && minr < mt) ++bad;
        }
      }
    }
  }
  std::printf("checks %ld bad %ld\n", checks, bad);
  return bad != 0;
}
