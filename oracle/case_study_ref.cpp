// case_study_ref.cpp — runs the reference's own case_study_heat
// (proj/src/case_study.cpp:171-290) and prints its result exactly.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile links this driver with the
// UNMODIFIED reference objects into oracle/_ref/case_study_ref.  It runs as
// its own process: the reference's iostream/filesystem code segfaults when
// loaded into a Python process next to numpy.
//
//   case_study_ref OUT_DIR EXTENT STEPS SAMPLE_EVERY MU SIGMA PATH THREADS [CK,CK,...]
//
// stdout: "series STEP CENTRE", "check STEP A1 A2 A3 R1 R2 R3", "final CENTRE",
// every double as a C99 hex float (%a) so the values round-trip bitwise.
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>

#include "tessera/case_study.hpp"

int main(int argc, char** argv) {
    if (argc < 9) {
        std::fprintf(stderr, "usage: %s OUT EXTENT STEPS SAMPLE_EVERY MU SIGMA PATH THREADS [CKS]\n",
                     argv[0]);
        return 2;
    }
    try {
        tessera::CaseStudyConfig cfg;
        cfg.extent = std::atoll(argv[2]);
        cfg.steps = std::atoll(argv[3]);
        cfg.sample_every = std::atoll(argv[4]);
        cfg.mu = std::strtod(argv[5], nullptr);
        cfg.sigma_cells = std::strtod(argv[6], nullptr);
        cfg.path = tessera::path_from_string(argv[7]);
        cfg.threads = std::atoi(argv[8]);
        cfg.checkpoints.clear();
        if (argc > 9) {
            std::istringstream vs(argv[9]);
            std::string tok;
            while (std::getline(vs, tok, ','))
                if (!tok.empty()) cfg.checkpoints.push_back(std::stoll(tok));
        }
        const tessera::CaseStudyResult r = tessera::case_study_heat(cfg, argv[1]);
        for (size_t i = 0; i < r.series_steps.size(); ++i)
            std::printf("series %lld %a\n", static_cast<long long>(r.series_steps[i]),
                        r.center_series[i]);
        for (size_t c = 0; c < r.checkpoint_steps.size(); ++c) {
            const auto& t = r.checkpoint_errors[c];
            std::printf("check %lld %a %a %a %a %a %a\n",
                        static_cast<long long>(r.checkpoint_steps[c]), t.abs_exceed_pct[0],
                        t.abs_exceed_pct[1], t.abs_exceed_pct[2], t.rel_exceed_pct[0],
                        t.rel_exceed_pct[1], t.rel_exceed_pct[2]);
        }
        std::printf("final %a\n", r.final_center);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
