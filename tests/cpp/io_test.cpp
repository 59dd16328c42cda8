// C++ drop-in, file I/O half (no GPU): written against the reference's own
// headers (stereotk/image.hpp, evaluate.hpp, error.hpp) and compiled against
// include/stereotk/; restates test_imaging.cpp:29-147 and
// test_evaluate.cpp:113-211 checks.  Exit code 0 = all checks passed.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "stereotk/error.hpp"
#include "stereotk/evaluate.hpp"
#include "stereotk/image.hpp"

using namespace stereotk;

static int failures = 0;
#define CHECK(c)                                                      \
    do {                                                              \
        if (!(c)) {                                                   \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                               \
        }                                                             \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<unsigned char> bytes(const std::string& p) {
    std::ifstream in(p, std::ios::binary);
    return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    GrayImage one(1, 1);
    one.data[0] = 255;
    save_gray(one, dir + "/one.pgm");
    const std::string want = "P5\n1 1\n255\n\xFF";
    CHECK(bytes(dir + "/one.pgm") == std::vector<unsigned char>(want.begin(), want.end()));

    GrayImage two(2, 1);
    two.data = {7, 9};
    save_gray(two, dir + "/c.pgm", {"scale 8"});
    std::vector<std::string> comments;
    CHECK(load_gray(dir + "/c.pgm", &comments).data == two.data);
    CHECK(comments.size() == 1 && comments[0] == "scale 8");

    RgbImage rgb(19, 33);
    for (std::size_t i = 0; i < rgb.data.size(); ++i) rgb.data[i] = static_cast<unsigned char>(i * 37 + 11);
    save_rgb(rgb, dir + "/rt.ppm");
    CHECK(load_image(dir + "/rt.ppm").data == rgb.data);
    save_rgb(rgb, dir + "/rt.png");
    const RgbImage back = load_image(dir + "/rt.png");
    CHECK(back.width == 19 && back.height == 33 && back.data == rgb.data);

    CHECK(throws<IoError>([&] { load_image(dir + "/no_such_file.ppm"); }));
    {
        std::ofstream(dir + "/garbage.ppm") << "this is not an image at all\n";
    }
    CHECK(throws<FormatError>([&] { load_image(dir + "/garbage.ppm"); }));

    GrayImage truth(4, 1);
    truth.data = {80, 0, 81, 88};
    save_gray(truth, dir + "/truth.pgm");
    const DisparityMap t = load_ground_truth(dir + "/truth.pgm", 16.0);
    CHECK((t.values == std::vector<std::int16_t>{5, -1, 5, 6}));
    CHECK(throws<ParamError>([&] { load_ground_truth(dir + "/truth.pgm", 0.0); }));

    DisparityMap d(3, 2);
    d.values = {0, 4, -1, 10, 31, 2};
    save_disparity(d, dir + "/disp.pgm", 8.0);
    CHECK(std::filesystem::exists(disparity_mask_path(dir + "/disp.pgm")));
    CHECK(load_disparity(dir + "/disp.pgm").values == d.values);
    CHECK(throws<ParamError>([&] { save_disparity(d, dir + "/o.pgm", 9.0); }));  // 31 * 9 > 255
    std::printf("%s (%d failures)\n", failures ? "FAIL" : "ok", failures);
    return failures ? 1 : 0;
}
