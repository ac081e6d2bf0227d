#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include "../include/phgrms_b200.h"
int main(int argc, char** argv) {
  int W = argc > 1 ? atoi(argv[1]) : 7, H = argc > 2 ? atoi(argv[2]) : 7;
  std::vector<uint8_t> img(W*H, 100), out(W*H);
  img[H/2*W + W/2] = 255;
  phg_params p{20, 1, 5, 3, 0};
  std::vector<phg_pass_stats> st(5); int it = 0;
  int rc = phg_denoise(img.data(), W, H, &p, 1, out.data(), st.data(), &it);
  printf("W=%d H=%d rc=%d err=%s it=%d rep0=%lld\n", W, H, rc, phg_last_error(), it, rc ? 0LL : (long long)st[0].replaced);
  return rc != 0;
}
