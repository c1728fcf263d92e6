// sanitize_main.cpp -- host-only driver for the ASan/UBSan build of the library's host half
// (decomposer, decomposition save/load/validation, distributed schedule, plan-builder argument
// validation).  Built and run by tests/test_sanitize.py with -fsanitize=address,undefined; no GPU is
// touched (plan creation is expected to stop at ARROW_E_CUDA without a device).
//   sanitize_main <csr file> <b> <tmpdir>
// csr file: int64 n, int64 nnz, int64 row_ptr[n+1], int32 col[nnz], float64 val[nnz] (little endian)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "arrow.h"

static int fails = 0;
#define CHECK(cond, msg)                                                  \
    do {                                                                  \
        if (!(cond)) {                                                    \
            std::fprintf(stderr, "FAIL %s: %s (%s)\n", msg, #cond, arrow_last_error()); \
            ++fails;                                                      \
        }                                                                 \
    } while (0)

int main(int argc, char **argv) {
    if (argc < 4) return 2;
    FILE *f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    int64_t n = 0, nnz = 0;
    if (std::fread(&n, 8, 1, f) != 1 || std::fread(&nnz, 8, 1, f) != 1) return 2;
    std::vector<int64_t> rp((size_t)n + 1);
    std::vector<int32_t> col((size_t)nnz);
    std::vector<double> val((size_t)nnz);
    if (std::fread(rp.data(), 8, rp.size(), f) != rp.size() || std::fread(col.data(), 4, col.size(), f) != col.size() ||
        std::fread(val.data(), 8, val.size(), f) != val.size())
        return 2;
    std::fclose(f);
    const int64_t b = std::atoll(argv[2]);
    const std::string tmp = argv[3];
    arrow_csr A{n, nnz, rp.data(), col.data(), val.data(), ARROW_F64};

    for (int band = 0; band <= 1; ++band) {
        arrow_decomposition d = nullptr;
        CHECK(arrow_decompose_ex(&A, b, 0, 4, 0, band, &d) == ARROW_OK, "decompose");
        int64_t dn = 0, db = 0, rn = 0;
        int32_t lv = 0;
        CHECK(arrow_decomposition_info(d, &dn, &db, &lv, &rn) == ARROW_OK && dn == n && rn == 0, "info");
        int64_t total = 0;
        for (int32_t i = 0; i < lv; ++i) {
            arrow_level_info_t li;
            CHECK(arrow_decomposition_level_info(d, i, &li) == ARROW_OK, "level_info");
            std::vector<int32_t> perm((size_t)li.rows), c((size_t)li.nnz);
            std::vector<int64_t> r((size_t)li.rows + 1);
            std::vector<double> v((size_t)li.nnz);
            CHECK(arrow_decomposition_export_level(d, i, perm.data(), r.data(), c.data(), v.data()) == ARROW_OK, "export");
            total += li.nnz;
        }
        CHECK(total == nnz, "levels partition the entries");
        // save / load round trip, then a corrupted copy must be rejected
        const std::string path = tmp + "/d" + std::to_string(band) + ".dec";
        CHECK(arrow_decomposition_save(d, path.c_str()) == ARROW_OK, "save");
        arrow_decomposition d2 = nullptr;
        CHECK(arrow_decomposition_load(path.c_str(), &d2) == ARROW_OK, "load");
        arrow_decomposition_destroy(d2);
        {
            FILE *g = std::fopen(path.c_str(), "r+b");
            std::fseek(g, 100, SEEK_SET);
            const unsigned char junk[8] = {0xff, 0xff, 0xff, 0x7f, 0x01, 0x02, 0x03, 0x04};
            std::fwrite(junk, 1, 8, g);
            std::fclose(g);
            arrow_decomposition d3 = nullptr;
            CHECK(arrow_decomposition_load(path.c_str(), &d3) != ARROW_OK && d3 == nullptr, "corrupt file rejected");
        }
        // distributed schedules (host only) for 2, 4, 8 ranks
        for (int G : {2, 4, 8}) {
            std::vector<int64_t> counts((size_t)lv * (4 * G + 4) + 8);
            for (int r = 0; r < G; ++r) {
                int64_t lohi[2] = {0, 0};
                CHECK(arrow_dist_schedule(d, G, r, 0, 0, lohi, counts.data()) == ARROW_OK, "dist_schedule");
            }
        }
        // plan creation without a device: ARROW_E_CUDA after the host half has run
        arrow_plan p = nullptr;
        const arrow_status ps = arrow_plan_create_from(d, nullptr, nullptr, &p);
        CHECK(ps == ARROW_E_CUDA && p == nullptr, "plan without a device");
        arrow_decomposition_destroy(d);
    }
    // home-set-aware levels (R25): decomposition, its homes, schedules for the homes' rank count (the
    // aligned path) and another one, save/load of format 3
    for (int homes : {2, 4}) {
        arrow_decomposition h = nullptr;
        CHECK(arrow_decompose_homes(&A, b, 0, 4, 0, 0, homes, 2, 0, &h) == ARROW_OK, "decompose_homes");
        int32_t hg = 0, hl = 0, lv = 0;
        std::vector<int64_t> ranges((size_t)homes + 1);
        CHECK(arrow_decomposition_homes(h, -1, &hg, &hl, ranges.data()) == ARROW_OK && hg == homes && hl == 2, "homes");
        CHECK(arrow_decomposition_info(h, nullptr, nullptr, &lv, nullptr) == ARROW_OK, "info");
        if (lv > 1) CHECK(arrow_decomposition_homes(h, 1, nullptr, nullptr, ranges.data()) == ARROW_OK, "home starts");
        for (int G : {homes, 3}) {
            std::vector<int64_t> counts((size_t)std::max(lv, 1) * (4 * G + 4) + 8);
            for (int r = 0; r < G; ++r) {
                int64_t lohi[2] = {0, 0};
                CHECK(arrow_dist_schedule(h, G, r, 0, 0, lohi, counts.data()) == ARROW_OK, "dist_schedule homes");
            }
        }
        const std::string path = tmp + "/h" + std::to_string(homes) + ".dec";
        CHECK(arrow_decomposition_save(h, path.c_str()) == ARROW_OK, "save homes");
        arrow_decomposition h2 = nullptr;
        CHECK(arrow_decomposition_load(path.c_str(), &h2) == ARROW_OK, "load homes");
        arrow_decomposition_destroy(h2);
        arrow_decomposition_destroy(h);
    }
    // level cap with residual, and the error paths of the argument validation
    arrow_decomposition d = nullptr;
    CHECK(arrow_decompose(&A, b, 1, 4, 1, &d) == ARROW_OK, "capped decomposition");
    arrow_decomposition_destroy(d);
    CHECK(arrow_decompose(&A, 1, 0, 4, 0, &d) == ARROW_E_INVALID_ARG, "b < 2");
    if (nnz > 1) {
        std::vector<int32_t> bad(col);
        bad[0] = (int32_t)n;  // out of range
        arrow_csr B{n, nnz, rp.data(), bad.data(), val.data(), ARROW_F64};
        CHECK(arrow_decompose(&B, b, 0, 4, 0, &d) == ARROW_E_BAD_CSR, "bad csr");
    }
    std::printf(fails ? "SANITIZE_FAIL %d\n" : "SANITIZE_OK\n", fails);
    return fails ? 1 : 0;
}
