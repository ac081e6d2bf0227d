#pragma once
// PGM file -> denoise -> PGM file with the file I/O overlapped with the
// host<->device copies (phg_denoise_pgm_file, include/phgrms_b200.h;
// SURVEY.md 8(f) f4).  The written file equals
//   save_pgm(out, denoise(load_pgm(in), params).image)
// of the reference (pgm.hpp:142-168, denoise.hpp:292-311); P2 input takes
// exactly that host path.

#include <string>
#include <vector>

#include "phgrms/denoise.hpp"
#include "phgrms/pgm.hpp"
#include "phgrms_b200.h"

namespace phgrms {

inline std::vector<PassStats> denoise_pgm_file(const std::string& in_path, const std::string& out_path,
                                               const DenoiseParams& params = DenoiseParams{}) {
    params.validate();
    {  // ASCII P2 input: the reference's codec on the host
        std::FILE* f = std::fopen(in_path.c_str(), "rb");
        if (!f) throw PgmError("cannot open " + in_path);
        const int c0 = std::fgetc(f), c1 = std::fgetc(f);
        std::fclose(f);
        if (c0 == 'P' && c1 == '2') {
            const auto res = denoise(load_pgm(in_path), params);
            save_pgm(out_path, res.image);
            return res.stats;
        }
    }
    const phg_params p = params.c();
    std::vector<phg_pass_stats> st(static_cast<std::size_t>(params.max_iterations));
    int iters = 0;
    const int rc = phg_denoise_pgm_file(in_path.c_str(), out_path.c_str(), &p, st.data(), &iters);
    if (rc == PHG_EINVAL) {
        const std::string msg = phg_last_error();
        if (msg.find("PGM") != std::string::npos || msg.find("cannot open") == 0 || msg.find("write failed") == 0)
            throw PgmError(msg);
    }
    detail::throw_on(rc);
    std::vector<PassStats> out;
    for (int i = 0; i < iters; ++i) out.push_back({st[i].iteration, st[i].flagged, st[i].replaced, st[i].elapsed_ms});
    return out;
}

}  // namespace phgrms
