// knn_b200_cli -- the reference CLI's `search` and `bench` subcommands on the
// B200 engine.
//
// Behaviour follows /root/reference/proj/tools/knn_cli.cpp (run_search, :66-96,
// the option table of main, :232-244) and accepts the same point/matrix files
// as src/csv.cpp (read_points_csv :85-94, read_matrix_csv :150-166); the file
// scanner and the output writer below are this engine's own (one in-memory
// pass, flat row-major table; stdio staging file + rename).  Same output
//   query_index,rank,ref_index,distance
// one row per (query, rank), replaced atomically through `<out>.tmp` + rename,
// and the same exit codes (main, :277-292): 0 success,
// 2 malformed input file ("error: line N: ..."), 3 contract violation
// (std::invalid_argument), 1 anything else, 2 for unknown options.
//
// `bench` mirrors run_grid / write_report_csv / write_report_json
// (src/bench.cpp:75-166, 207-232) for the brute-force method: per (n, d) cell
// uniform points from mt19937_64 seeded derive_seed(seed, n, d, 0 | 1)
// (include/knn/rng.hpp), bf_knn timed `--reps` times (median; first rep is
// warm-up from 4 reps on), the time budget, and the report schema
//   method,n,d,k,seconds,dist_evals,seed
// `kdt` rows are not available (the kd-tree is outside this engine): asking
// for them is a contract error (exit 3).
//
// Differences a caller can see: the search runs on the GPU in FP32 (distances
// are printed as the shortest decimal of the FP32 value, so the reference's
// CLI test fixture prints identically: 0.1 / 0.9 / 1.9), and `--method kdtree`
// runs the same exact search (the kd-tree reports the same neighbours,
// test_cli.cpp:70-75); --workers / --chunk-size / --leaf-size are accepted
// and do not change results.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <system_error>
#include <vector>

#include "knn_b200/bruteforce.hpp"

namespace {

struct CsvError : std::runtime_error {  // csv.hpp:16-25
    CsvError(const std::string& message, std::size_t line)
        : std::runtime_error("line " + std::to_string(line) + ": " + message) {}
};

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- point files -----------------------------------------------------------
// One pass over the whole file held in memory: a small scanner walks the bytes,
// cutting fields at ',' and records at '\n', and converts each field as soon as
// it is cut, so the table is a flat row-major vector from the start (no per-row
// string copies).  Accepted input is the reference's (src/csv.cpp): blank
// lines and lines whose first non-blank character is '#' are skipped, spaces,
// tabs and a trailing '\r' around a field are ignored, and every record must
// have as many fields as the first one.  Errors name the 1-based file line.
struct NumericTable {
    std::vector<double> values;  // row-major
    std::size_t cols = 0, rows = 0;
    std::size_t last_line = 0;   // file line of the last record
};

bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

double field_value(const char* b, const char* e, std::size_t line) {
    while (b < e && is_blank(*b)) ++b;
    while (e > b && is_blank(e[-1])) --e;
    double v = 0.0;
    const std::from_chars_result r = std::from_chars(b, e, v);
    if (r.ec != std::errc{} || r.ptr != e)
        throw CsvError("cannot parse '" + std::string(b, e) + "' as a number", line);
    return v;
}

NumericTable scan_numeric_file(const std::filesystem::path& path) {
    std::string text;
    {
        std::FILE* f = std::fopen(path.c_str(), "rb");
        if (f == nullptr) throw std::runtime_error("cannot open '" + path.string() + "'");
        char chunk[1 << 16];
        for (std::size_t got; (got = std::fread(chunk, 1, sizeof chunk, f)) > 0;) text.append(chunk, got);
        std::fclose(f);
    }
    NumericTable t;
    const char* p = text.data();
    const char* const end = p + text.size();
    for (std::size_t line = 1; p < end; ++line) {
        const char* eol = static_cast<const char*>(std::memchr(p, '\n', static_cast<std::size_t>(end - p)));
        if (eol == nullptr) eol = end;
        const char* first = p;
        while (first < eol && is_blank(*first)) ++first;
        if (first < eol && *first != '#') {  // a record
            std::size_t width = 0;
            for (const char* f = p;; ++width) {
                const char* comma = std::find(f, eol, ',');
                t.values.push_back(field_value(f, comma, line));
                if (comma == eol) break;
                f = comma + 1;
            }
            ++width;
            if (t.rows == 0) t.cols = width;
            else if (width != t.cols)
                throw CsvError("expected " + std::to_string(t.cols) + " fields, got " + std::to_string(width),
                               line);
            ++t.rows;
            t.last_line = line;
        }
        p = eol + (eol < end ? 1 : 0);
    }
    if (t.rows == 0) throw CsvError("no data rows in " + path.string(), 0);
    return t;
}

knn_b200::PointSet read_points_csv(const std::filesystem::path& path) {
    NumericTable t = scan_numeric_file(path);
    return knn_b200::PointSet(t.rows, t.cols, std::move(t.values));
}

std::vector<double> read_matrix_csv(const std::filesystem::path& path, std::size_t& dim) {
    NumericTable t = scan_numeric_file(path);
    if (t.rows != t.cols)
        throw CsvError("matrix must be square, got " + std::to_string(t.rows) + "x" + std::to_string(t.cols),
                       t.last_line);
    dim = t.cols;
    return std::move(t.values);
}

knn_b200::Metric parse_metric(const std::string& spec) {
    static constexpr std::string_view kMaha = "mahalanobis:";
    if (spec.size() > kMaha.size() && spec.compare(0, kMaha.size(), kMaha) == 0) {
        std::size_t dim = 0;
        std::vector<double> cov = read_matrix_csv(spec.substr(kMaha.size()), dim);
        return knn_b200::Metric::mahalanobis(dim, std::move(cov));
    }
    using Factory = knn_b200::Metric (*)();
    static const std::pair<std::string_view, Factory> kPlain[] = {
        {"euclidean", &knn_b200::Metric::euclidean},
        {"manhattan", &knn_b200::Metric::manhattan},
        {"chebyshev", &knn_b200::Metric::chebyshev},
    };
    for (const auto& [name, make] : kPlain)
        if (spec == name) return make();
    throw UsageError("--metric: expected euclidean, manhattan, chebyshev or mahalanobis:PATH");
}

// stdout when no path is given; otherwise the whole text goes to "<path>.tmp",
// which then replaces <path> in one rename (readers never see a partial file)
void emit(const std::string& path, const std::string& text) {
    if (path.empty()) {
        std::fwrite(text.data(), 1, text.size(), stdout);
        std::fflush(stdout);
        return;
    }
    const std::string staging = path + ".tmp";
    std::FILE* f = std::fopen(staging.c_str(), "wb");
    if (f == nullptr) throw std::runtime_error("cannot open '" + staging + "' for writing");
    const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
    if (std::fclose(f) != 0 || !ok) throw std::runtime_error("cannot write '" + staging + "'");
    std::error_code ec;
    std::filesystem::rename(staging, path, ec);
    if (ec) throw std::runtime_error("cannot replace '" + path + "': " + ec.message());
}

std::string format_distance(double d) {  // the FP32 value's shortest decimal
    char buf[32];
    const auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), static_cast<float>(d));
    return std::string(buf, ptr);
}

template <typename T>
T parse_number(const std::string& opt, const std::string& v) {
    T out{};
    const auto [ptr, ec] = std::from_chars(v.data(), v.data() + v.size(), out);
    if (ec != std::errc{} || ptr != v.data() + v.size())
        throw UsageError(opt + ": '" + v + "' is not a valid number");
    return out;
}

int run_search(int argc, char** argv) {
    std::string ref_path, query_path, out_path, metric = "euclidean", method = "bf";
    std::size_t k = 0, chunk_size = 1024;
    bool have_k = false;
    for (int i = 2; i < argc; ++i) {
        const std::string opt = argv[i];
        if (i + 1 >= argc) throw UsageError(opt + ": missing value");
        const std::string val = argv[++i];
        if (opt == "--ref") ref_path = val;
        else if (opt == "--query") query_path = val;
        else if (opt == "--out") out_path = val;
        else if (opt == "--metric") metric = val;
        else if (opt == "--method") method = val;
        else if (opt == "--k") k = parse_number<std::size_t>(opt, val), have_k = true;
        else if (opt == "--chunk-size") chunk_size = parse_number<std::size_t>(opt, val);
        else if (opt == "--workers") parse_number<unsigned>(opt, val);
        else if (opt == "--leaf-size") parse_number<std::size_t>(opt, val);
        else throw UsageError("The following argument was not expected: " + opt);
    }
    if (ref_path.empty()) throw UsageError("--ref is required");
    if (query_path.empty()) throw UsageError("--query is required");
    if (!have_k) throw UsageError("--k is required");
    if (method != "bf" && method != "kdtree") throw UsageError("--method: expected bf or kdtree");

    const knn_b200::PointSet refs = read_points_csv(ref_path);
    const knn_b200::PointSet queries = read_points_csv(query_path);
    const knn_b200::Metric m = parse_metric(metric);
    knn_b200::BfConfig config;
    config.chunk_size = chunk_size;
    const knn_b200::NeighborTable table = knn_b200::bf_knn(queries, refs, k, m, config);

    std::ostringstream out;
    out << "query_index,rank,ref_index,distance\n";
    for (std::size_t i = 0; i < table.query_count(); ++i) {
        const auto row = table.row(i);
        for (std::size_t r = 0; r < row.size(); ++r)
            out << i << ',' << r << ',' << row[r].index << ',' << format_distance(row[r].distance)
                << '\n';
    }
    emit(out_path, out.str());
    return 0;
}

// include/knn/rng.hpp: splitmix64, derive_seed, next_unit
std::uint64_t splitmix64(std::uint64_t& state) {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

std::uint64_t derive_seed(std::uint64_t master, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
    std::uint64_t state = master;
    std::uint64_t out = splitmix64(state);
    state ^= a * 0x9e3779b97f4a7c15ULL;
    out ^= splitmix64(state);
    state ^= b * 0xbf58476d1ce4e5b9ULL;
    out ^= splitmix64(state);
    state ^= c * 0x94d049bb133111ebULL;
    out ^= splitmix64(state);
    return out;
}

knn_b200::PointSet generate_uniform(std::size_t n, std::size_t d, std::uint64_t seed) {
    std::mt19937_64 gen(seed);  // bench.cpp:39-46
    std::vector<double> data(n * d);
    for (double& v : data) v = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    return knn_b200::PointSet(n, d, std::move(data));
}

std::vector<std::size_t> parse_list(const std::string& opt, const std::string& v) {
    std::vector<std::size_t> out;
    std::size_t start = 0;
    while (true) {
        const std::size_t comma = v.find(',', start);
        out.push_back(parse_number<std::size_t>(opt, v.substr(start, comma - start)));
        if (comma == std::string::npos) break;
        start = comma + 1;
    }
    return out;
}

std::vector<std::string> parse_methods(const std::string& v) {  // bench.cpp:27-31 names
    std::vector<std::string> out;
    std::size_t start = 0;
    while (true) {
        const std::size_t comma = v.find(',', start);
        std::string name = v.substr(start, comma - start);
        if (name == "kdtree") name = "kdt";
        if (name != "bf" && name != "kdt")
            throw std::invalid_argument("unknown method '" + name + "', expected bf or kdt");
        out.push_back(name);
        if (comma == std::string::npos) break;
        start = comma + 1;
    }
    return out;
}

std::string format_double(double value) {  // csv.cpp:172-176
    char buf[32];
    const auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), value);
    return std::string(buf, ptr);
}

int run_bench(int argc, char** argv) {
    std::vector<std::size_t> n_values{1200, 2400}, d_values{8, 16, 32, 64, 80, 96};  // default_grid
    std::string metric = "euclidean", out_path, json_path, methods = "bf";
    std::size_t k = 20, reps = 3;
    std::uint64_t seed = 0;
    double budget = 120.0;
    for (int i = 2; i < argc; ++i) {
        const std::string opt = argv[i];
        if (i + 1 >= argc) throw UsageError(opt + ": missing value");
        const std::string val = argv[++i];
        if (opt == "--grid") {
            if (val != "default") throw UsageError("--grid: the only named grid is 'default'");
        } else if (opt == "--n-values") n_values = parse_list(opt, val);
        else if (opt == "--d-values") d_values = parse_list(opt, val);
        else if (opt == "--methods") methods = val;
        else if (opt == "--metric") metric = val;
        else if (opt == "--k") k = parse_number<std::size_t>(opt, val);
        else if (opt == "--reps") reps = parse_number<std::size_t>(opt, val);
        else if (opt == "--seed") seed = parse_number<std::uint64_t>(opt, val);
        else if (opt == "--workers") parse_number<unsigned>(opt, val);
        else if (opt == "--time-budget") budget = parse_number<double>(opt, val);
        else if (opt == "--out") out_path = val;
        else if (opt == "--json") json_path = val;
        else throw UsageError("The following argument was not expected: " + opt);
    }
    for (const std::string& mth : parse_methods(methods))
        if (mth != "bf")
            throw std::invalid_argument("method '" + mth +
                                        "' is not available on the B200 engine (bf only)");
    if (reps == 0) throw std::invalid_argument("run_grid: repetitions must be >= 1");
    for (std::size_t n : n_values)
        if (k > n)
            throw std::invalid_argument("run_grid: k = " + std::to_string(k) +
                                        " exceeds cell size n = " + std::to_string(n));
    const knn_b200::Metric m = parse_metric(metric);

    std::ostringstream csv, json;
    csv << "method,n,d,k,seconds,dist_evals,seed\n";
    json << "{\n  \"environment\": \"knn_b200 engine (B200), metric " << metric
         << ", points uniform [0,1)^d\",\n  \"rows\": [";
    bool first = true;
    for (std::size_t n : n_values)
        for (std::size_t d : d_values) {
            const knn_b200::PointSet refs = generate_uniform(n, d, derive_seed(seed, n, d, 0));
            const knn_b200::PointSet queries = generate_uniform(n, d, derive_seed(seed, n, d, 1));
            knn_b200::BfConfig cfg;
            cfg.count_distance_evals = true;
            std::vector<double> times;
            std::uint64_t evals = 0;
            bool skipped = false;
            for (std::size_t rep = 0; rep < reps; ++rep) {
                knn_b200::SearchStats stats;
                const auto t0 = std::chrono::steady_clock::now();
                (void)knn_b200::bf_knn(queries, refs, k, m, cfg, &stats);
                times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
                evals = stats.distance_evals;
                if (rep == 0 && times[0] > budget) {
                    skipped = true;
                    break;
                }
            }
            double seconds = NAN;
            if (!skipped) {
                std::vector<double> t(times.begin() + (reps >= 4 ? 1 : 0), times.end());
                std::sort(t.begin(), t.end());
                const std::size_t mid = t.size() / 2;
                seconds = t.size() % 2 ? t[mid] : 0.5 * (t[mid - 1] + t[mid]);
            }
            std::cerr << "bf n=" << n << " d=" << d << " k=" << k
                      << (skipped ? " skipped (over time budget)" : " seconds=" + format_double(seconds))
                      << " dist_evals=" << evals << '\n';
            csv << "bf," << n << ',' << d << ',' << k << ',' << (skipped ? "NA" : format_double(seconds))
                << ',' << evals << ',' << seed << '\n';
            json << (first ? "" : ",") << "\n    {\"method\": \"bf\", \"n\": " << n << ", \"d\": " << d
                 << ", \"k\": " << k << ", \"dist_evals\": " << evals << ", \"seed\": " << seed
                 << ", \"skipped\": " << (skipped ? "true" : "false") << ", \"seconds\": "
                 << (skipped ? "null" : format_double(seconds)) << "}";
            first = false;
        }
    json << "\n  ]\n}\n";
    emit(out_path, csv.str());
    if (!json_path.empty()) emit(json_path, json.str());
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const std::string cmd = argc >= 2 ? argv[1] : "";
        if (cmd == "search") return run_search(argc, argv);
        if (cmd == "bench") return run_bench(argc, argv);
        throw UsageError("usage: knn_b200_cli search --ref R.csv --query Q.csv --k K "
                         "[--metric M] [--method bf|kdtree] [--out OUT.csv]\n"
                         "       knn_b200_cli bench [--grid default] [--n-values N,..] "
                         "[--d-values D,..] [--k K] [--reps R] [--seed S] [--out OUT.csv] "
                         "[--json OUT.json]");
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const CsvError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
