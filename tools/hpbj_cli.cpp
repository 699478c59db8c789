// hpbj_cli — the reference benchmark harness (tools/bjgmres_cli.cpp) on the
// B200 solver: same subcommands, options, JSON report schema, history CSV and
// bench table, so scripts written against the reference
// harness run unchanged. Built by __graft_entry__.build() into
// paper_2509_09139_b200/lib/hpbj_cli (links libhpbj.so through
// include/bjgmres_b200.hpp).
//
//   hpbj_cli solve --matrix A.mtx [--rhs ones|axones|random:SEED|file:PATH]
//            [--precond block-jacobi|ilu0|none] [--blocks S] [--restart M] [--tol T]
//            [--max-restarts R] [--precision hybrid] [--eps-pivot E] [--neumann-order K]
//            [--partition-file P] [--absolute-tol] [--report R.json]
//            [--history H.csv]
//   hpbj_cli bench --specs specs.json [--repetitions K] [--out table.csv]
//   hpbj_cli partition --matrix A.mtx --blocks S --out P.txt
//
// Differences from the reference harness: the device path
// runs block Jacobi in the north star's precision mix only, so --precision
// defaults to "hybrid" for it and "double" is rejected there (ILU(0) and none
// default to "double", like the reference, and run in FP64); --ritz is
// rejected.
// Exit codes: 0 converged, 2 not converged (solve), 1 error.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "bjgmres_b200.hpp"
#include "hpbj.h"

using namespace bjgmres_b200;

namespace {

// ---------------------------------------------------------------------------
// Minimal JSON value (parse for bench specs, emit for reports).
struct Json {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<Json> arr;
    std::vector<std::pair<std::string, Json>> obj;
    const Json* get(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct JsonParser {
    const std::string& s;
    size_t i = 0;
    explicit JsonParser(const std::string& t) : s(t) {}
    [[noreturn]] void err(const std::string& m) {
        throw std::runtime_error("specs JSON: " + m + " at offset " + std::to_string(i));
    }
    void ws() {
        while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
    }
    Json value() {
        ws();
        if (i >= s.size()) err("unexpected end");
        const char c = s[i];
        Json v;
        if (c == '{') {
            v.kind = Json::Obj;
            ++i;
            ws();
            if (i < s.size() && s[i] == '}') {
                ++i;
                return v;
            }
            for (;;) {
                ws();
                if (i >= s.size() || s[i] != '"') err("expected key");
                std::string k = string();
                ws();
                if (i >= s.size() || s[i] != ':') err("expected ':'");
                ++i;
                v.obj.emplace_back(k, value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == '}') {
                    ++i;
                    return v;
                }
                err("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = Json::Arr;
            ++i;
            ws();
            if (i < s.size() && s[i] == ']') {
                ++i;
                return v;
            }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == ']') {
                    ++i;
                    return v;
                }
                err("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = Json::Str;
            v.str = string();
            return v;
        }
        if (s.compare(i, 4, "true") == 0) {
            i += 4;
            v.kind = Json::Bool;
            v.b = true;
            return v;
        }
        if (s.compare(i, 5, "false") == 0) {
            i += 5;
            v.kind = Json::Bool;
            return v;
        }
        if (s.compare(i, 4, "null") == 0) {
            i += 4;
            return v;
        }
        char* end = nullptr;
        v.num = std::strtod(s.c_str() + i, &end);
        if (end == s.c_str() + i) err("unexpected character");
        i = end - s.c_str();
        v.kind = Json::Num;
        return v;
    }
    std::string string() {
        ++i;  // opening quote
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                ++i;
                if (i >= s.size()) err("bad escape");
                const char e = s[i];
                if (e == 'n') out += '\n';
                else if (e == 't') out += '\t';
                else if (e == 'r') out += '\r';
                else if (e == 'b') out += '\b';
                else if (e == 'f') out += '\f';
                else if (e == 'u') {
                    if (i + 4 >= s.size()) err("bad \\u escape");
                    const unsigned cp = (unsigned)std::stoul(s.substr(i + 1, 4), nullptr, 16);
                    if (cp < 0x80) out += (char)cp;  // specs are ASCII paths/keywords
                    else out += '?';
                    i += 4;
                } else out += e;
                ++i;
            } else {
                out += s[i++];
            }
        }
        if (i >= s.size()) err("unterminated string");
        ++i;
        return out;
    }
};

std::string jstr(const std::string& v) {
    std::string o = "\"";
    for (const char c : v) {
        if (c == '"' || c == '\\') o += '\\', o += c;
        else if (c == '\n') o += "\\n";
        else if ((unsigned char)c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", (unsigned char)c);
            o += b;
        } else o += c;
    }
    return o + "\"";
}
std::string jnum(double v) {
    if (!std::isfinite(v)) return "null";
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}
std::string jint(long long v) { return std::to_string(v); }
std::string jbool(bool v) { return v ? "true" : "false"; }

// ---------------------------------------------------------------------------
struct RunSpec {  // bjgmres_cli.cpp:29-45, with this build's precision default
    std::string matrix_path;
    std::string rhs_mode = "axones";
    std::string precond = "block-jacobi";
    index_t blocks = 16;
    index_t restart_m = 50;
    double tol = 1e-8;
    index_t max_restarts = 40;
    std::string precision;  // "" = this build's default: hybrid for block-jacobi, double otherwise
    double eps_pivot = 1e-10;
    int neumann_order = 0;
    std::string partition_file;
    bool absolute_tol = false;
    bool ritz = false;
    std::string report_path;
    std::string history_path;
};

struct RunResult {
    std::string matrix_name;
    index_t n = 0, nnz = 0;
    double setup_ms = 0.0, solve_ms = 0.0;
    SolveReport report;
    std::vector<double> x;
    std::vector<index_t> block_dim, block_nnz, block_pert;
    std::vector<double> block_cond, block_ebound;
};

std::string matrix_name_of(const std::string& path) {
    std::string name = path;
    const size_t slash = name.find_last_of("/\\");
    if (slash != std::string::npos) name = name.substr(slash + 1);
    const size_t dot = name.find_last_of('.');
    if (dot != std::string::npos && dot > 0) name = name.substr(0, dot);
    return name;
}

SparseMatrix read_matrix(const std::string& path, index_t* ncols_out = nullptr) {
    int64_t nr = 0, nc = 0;
    int64_t *rp = nullptr, *ci = nullptr;
    double* v = nullptr;
    if (hpbj_mm_read(path.c_str(), &nr, &nc, &rp, &ci, &v) != HPBJ_OK) throw std::runtime_error(hpbj_last_error(nullptr));
    std::vector<index_t> r(rp, rp + nr + 1), c(ci, ci + rp[nr]);
    std::vector<double> vv(v, v + rp[nr]);
    hpbj_free(rp);
    hpbj_free(ci);
    hpbj_free(v);
    if (nr != nc)
        throw std::runtime_error("matrix must be square, got " + std::to_string(nr) + "x" + std::to_string(nc));
    if (ncols_out) *ncols_out = nc;
    return SparseMatrix(nr, nc, std::move(r), std::move(c), std::move(vv));
}

// SplitMix64 in [-1, 1) (the reference's seeded_rhs, bjgmres_cli.cpp:67-79)
std::vector<double> seeded_rhs(index_t n, std::uint64_t seed) {
    std::vector<double> b(n);
    std::uint64_t st = seed;
    for (double& v : b) {
        std::uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z = z ^ (z >> 31);
        v = static_cast<double>(z >> 11) * 0x1p-53 * 2.0 - 1.0;
    }
    return b;
}

std::vector<double> make_rhs(const RunSpec& spec, const SparseMatrix& a) {
    const index_t n = a.rows();
    if (spec.rhs_mode == "ones") return std::vector<double>(n, 1.0);
    if (spec.rhs_mode == "axones") {  // spmv<double>(A, 1): row sums, left to right
        std::vector<double> b(n);
        const auto rs = a.row_starts();
        const auto v = a.values();
        for (index_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (index_t k = rs[i]; k < rs[i + 1]; ++k) s += v[k] * 1.0;
            b[i] = s;
        }
        return b;
    }
    if (spec.rhs_mode.rfind("random:", 0) == 0) return seeded_rhs(n, std::stoull(spec.rhs_mode.substr(7)));
    if (spec.rhs_mode.rfind("file:", 0) == 0) {
        const std::string path = spec.rhs_mode.substr(5);
        std::ifstream in(path);
        if (!in) throw std::runtime_error("cannot open rhs file: " + path);
        std::vector<double> b;
        double v;
        while (in >> v) b.push_back(v);
        if ((index_t)b.size() != n)
            throw std::runtime_error("rhs file length " + std::to_string(b.size()) +
                                     " does not match matrix dimension " + std::to_string(n));
        return b;
    }
    throw std::runtime_error("unknown rhs mode: " + spec.rhs_mode);
}

Partition import_partition_file(const std::string& path, index_t n, index_t s) {  // partition.cpp:145-172
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open partition file: " + path);
    std::vector<index_t> asg;
    std::string line;
    long line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        std::istringstream ls(line);
        index_t b;
        if (!(ls >> b)) {
            if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
            throw std::runtime_error("partition file: line " + std::to_string(line_no) + ": malformed");
        }
        if (b < 0 || b >= s)
            throw std::out_of_range("partition file: line " + std::to_string(line_no) + ": block index " +
                                    std::to_string(b) + " out of range");
        asg.push_back(b);
    }
    if ((index_t)asg.size() != n)
        throw std::runtime_error("partition file: expected " + std::to_string(n) + " lines, got " +
                                 std::to_string(asg.size()));
    return partition_from_assignment(std::move(asg), s);
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

RunResult run_spec(const RunSpec& spec) {  // bjgmres_cli.cpp:112-168
    RunResult out;
    out.matrix_name = matrix_name_of(spec.matrix_path);
    SparseMatrix a = read_matrix(spec.matrix_path);
    out.n = a.rows();
    out.nnz = a.nnz();
    const auto t_setup = std::chrono::steady_clock::now();
    if (spec.precision == "hybrid") a.materialize_low();  // bjgmres_cli.cpp:126
    GmresConfig cfg;
    cfg.restart_m = spec.restart_m;
    cfg.tol = spec.tol;
    cfg.max_restarts = spec.max_restarts;
    cfg.absolute_tol = spec.absolute_tol;
    cfg.policy.mode = spec.precision == "hybrid" ? PrecisionMode::Hybrid : PrecisionMode::DoubleOnly;
    if (spec.precond != "block-jacobi") {  // bjgmres_cli.cpp:128-131, 152-154
        Preconditioner p = Preconditioner::identity(a.rows());
        if (spec.precond == "ilu0") p = Preconditioner::from_ilu0(a);
        else if (spec.precond != "none") throw std::runtime_error("unknown preconditioner: " + spec.precond);
        out.setup_ms = ms_since(t_setup);
        const std::vector<double> b = make_rhs(spec, a);
        const auto t_solve = std::chrono::steady_clock::now();
        SolveResult sr = hybrid_restart_gmres(a, p, b, cfg);
        out.solve_ms = ms_since(t_solve);
        out.report = std::move(sr.report);
        out.x = std::move(sr.x);
        return out;
    }
    Partition part;
    if (!spec.partition_file.empty()) part = import_partition_file(spec.partition_file, a.rows(), spec.blocks);
    else part = partition_graph(a, spec.blocks, 0.1);
    BlockJacobiOptions opts;
    opts.eps_pivot = spec.eps_pivot;
    opts.neumann_order = spec.neumann_order;
    opts.policy.mode = cfg.policy.mode;
    Preconditioner p = Preconditioner::block_jacobi(a, std::move(part), opts);
    // with_cond_estimates defaults to true in the reference (preconditioner.hpp:37):
    // the estimates are part of its setup time
    const auto& stats = p.block_jacobi_data()->stats;
    out.setup_ms = ms_since(t_setup);
    for (const auto& st : stats) {
        out.block_nnz.push_back(st.block_nnz);
        out.block_dim.push_back(st.block_dim);
        out.block_pert.push_back(st.perturbation_count);
        out.block_cond.push_back(st.cond_estimate);
        out.block_ebound.push_back(st.error_bound);
    }
    const std::vector<double> b = make_rhs(spec, a);
    const auto t_solve = std::chrono::steady_clock::now();
    SolveResult sr = hybrid_restart_gmres(a, p, b, cfg);
    out.solve_ms = ms_since(t_solve);
    out.report = std::move(sr.report);
    out.x = std::move(sr.x);
    return out;
}

std::string config_json(const RunSpec& s) {
    std::string o = "{\n    \"matrix\": " + jstr(s.matrix_path) + ",\n    \"rhs\": " + jstr(s.rhs_mode) +
                    ",\n    \"precond\": " + jstr(s.precond) + ",\n    \"blocks\": " + jint(s.blocks) +
                    ",\n    \"restart\": " + jint(s.restart_m) + ",\n    \"tol\": " + jnum(s.tol) +
                    ",\n    \"max_restarts\": " + jint(s.max_restarts) + ",\n    \"precision\": " + jstr(s.precision) +
                    ",\n    \"eps_pivot\": " + jnum(s.eps_pivot) + ",\n    \"neumann_order\": " + jint(s.neumann_order) +
                    ",\n    \"partition_file\": " + (s.partition_file.empty() ? "null" : jstr(s.partition_file)) +
                    ",\n    \"absolute_tol\": " + jbool(s.absolute_tol) + ",\n    \"ritz\": " + jbool(s.ritz) + "\n  }";
    return o;
}

std::string report_json(const RunSpec& spec, const RunResult& r) {  // bjgmres_cli.cpp:189-214 schema
    std::string o = "{\n  \"matrix\": {\"name\": " + jstr(r.matrix_name) + ", \"n\": " + jint(r.n) +
                    ", \"nnz\": " + jint(r.nnz) + "},\n  \"config\": " + config_json(spec) + ",\n  \"result\": {" +
                    "\"converged\": " + jbool(r.report.converged) + ", \"iterations\": " +
                    jint(r.report.total_iterations) + ", \"restarts\": " + jint(r.report.restarts) +
                    ", \"final_residual\": " + jnum(r.report.final_residual) + ", \"setup_ms\": " + jnum(r.setup_ms) +
                    ", \"solve_ms\": " + jnum(r.solve_ms) + "},\n  \"preconditioner\": {\"blocks\": [";
    for (size_t b = 0; b < r.block_dim.size(); ++b) {
        o += (b ? ",\n    " : "\n    ");
        o += "{\"dim\": " + jint(r.block_dim[b]) + ", \"nnz\": " + jint(r.block_nnz[b]) + ", \"perturbations\": " +
             jint(r.block_pert[b]) + ", \"cond_estimate\": " + jnum(r.block_cond[b]) + ", \"error_bound\": " +
             jnum(r.block_ebound[b]) + "}";
    }
    o += "\n  ]}\n}\n";
    return o;
}

void write_history_csv(const std::string& path, const SolveReport& rep) {  // bjgmres_cli.cpp:216-225
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open history file: " + path);
    out << "restart_cycle,global_iteration,relative_residual\n";
    char buf[64];
    for (const HistoryPoint& h : rep.residual_history) {
        std::snprintf(buf, sizeof buf, "%.17g", h.relative_residual);
        out << h.cycle << "," << h.iteration << "," << buf << "\n";
    }
}

void print_summary(const RunResult& r) {
    std::printf("%s: n=%lld nnz=%lld\n", r.matrix_name.c_str(), (long long)r.n, (long long)r.nnz);
    std::printf("  converged=%s iterations=%lld restarts=%lld final_residual=%.3e\n",
                r.report.converged ? "true" : "false", (long long)r.report.total_iterations,
                (long long)r.report.restarts, r.report.final_residual);
    std::printf("  setup=%.2f ms  solve=%.2f ms\n", r.setup_ms, r.solve_ms);
}

double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 == 1 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

// the option checks the reference applies (bjgmres_cli.cpp:414-433), plus
// this build's restrictions
std::string check_spec(RunSpec& s, bool blocks_set, bool part_set, bool neu_set, bool eps_set) {
    if (s.precond != "block-jacobi") {
        if (blocks_set) return "--blocks requires --precond block-jacobi";
        if (part_set) return "--partition-file requires --precond block-jacobi";
        if (neu_set) return "--neumann-order requires --precond block-jacobi";
        if (eps_set) return "--eps-pivot requires --precond block-jacobi";
    }
    if (s.precision.empty()) s.precision = s.precond == "block-jacobi" ? "hybrid" : "double";
    if (s.precision != "double" && s.precision != "hybrid") return "unknown precision: " + s.precision;
    if (s.precond == "block-jacobi" && s.precision == "double")
        return "precision 'double' with block-jacobi is not implemented on the GPU path (FP32 block factors)";
    if (s.ritz) return "--ritz is not implemented on the GPU path";
    if (s.blocks < 1 || s.restart_m < 1 || s.max_restarts < 1 || s.tol <= 0.0) return "numeric flags out of range";
    return "";
}

RunSpec spec_from_json(const Json& j) {  // bjgmres_cli.cpp:235-250
    RunSpec s;
    const Json* m = j.get("matrix");
    if (!m || m->kind != Json::Str) throw std::runtime_error("spec needs a \"matrix\" string");
    s.matrix_path = m->str;
    auto str = [&](const char* k, std::string& dst) {
        if (const Json* v = j.get(k); v && v->kind == Json::Str) dst = v->str;
    };
    auto num = [&](const char* k, auto& dst) {
        if (const Json* v = j.get(k); v && v->kind == Json::Num) dst = static_cast<std::decay_t<decltype(dst)>>(v->num);
    };
    str("rhs", s.rhs_mode);
    str("precond", s.precond);
    num("blocks", s.blocks);
    num("restart", s.restart_m);
    num("tol", s.tol);
    num("max_restarts", s.max_restarts);
    str("precision", s.precision);
    num("eps_pivot", s.eps_pivot);
    num("neumann_order", s.neumann_order);
    str("partition_file", s.partition_file);
    if (const Json* v = j.get("absolute_tol"); v && v->kind == Json::Bool) s.absolute_tol = v->b;
    return s;
}

int cmd_bench(const std::string& specs_path, int repetitions, const std::string& out_csv) {  // :252-347
    std::ifstream in(specs_path);
    if (!in) {
        std::cerr << "error: cannot open specs file: " << specs_path << "\n";
        return 1;
    }
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    Json specs;
    try {
        JsonParser jp(text);
        specs = jp.value();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    if (specs.kind != Json::Arr || specs.arr.empty()) {
        std::cerr << "error: specs file must hold a non-empty JSON array\n";
        return 1;
    }
    struct Row {
        std::string name;
        index_t n, nnz, iterations;
        double setup_ms, solve_ms, final_residual;
        bool converged;
    };
    std::vector<Row> rows;
    for (const Json& j : specs.arr) {
        try {
            RunSpec spec = spec_from_json(j);
            const std::string bad = check_spec(spec, false, false, false, false);
            if (!bad.empty()) throw std::runtime_error(bad);
            std::vector<double> st, sv;
            RunResult last;
            for (int rep = 0; rep < repetitions; ++rep) {
                last = run_spec(spec);
                st.push_back(last.setup_ms);
                sv.push_back(last.solve_ms);
            }
            rows.push_back({last.matrix_name, last.n, last.nnz, last.report.total_iterations, median(st), median(sv),
                            last.report.final_residual, last.report.converged});
        } catch (const std::exception& e) {
            std::cerr << "warning: skipping spec (" << e.what() << ")\n";
        }
    }
    if (rows.empty()) {
        std::cerr << "error: every spec failed\n";
        return 1;
    }
    std::printf("%-16s %8s %9s %8s %12s %11s %6s %5s %13s\n", "matrix", "n", "nnz", "nnz/row", "setup(ms)",
                "solve(ms)", "iter", "conv", "residual");
    for (const Row& r : rows)
        std::printf("%-16s %8lld %9lld %8.2f %12.2f %11.2f %6lld %5s %13.3e\n", r.name.c_str(), (long long)r.n,
                    (long long)r.nnz, (double)r.nnz / (double)r.n, r.setup_ms, r.solve_ms, (long long)r.iterations,
                    r.converged ? "yes" : "no", r.final_residual);
    if (!out_csv.empty()) {
        std::ofstream csv(out_csv);
        if (!csv) {
            std::cerr << "error: cannot open " << out_csv << "\n";
            return 1;
        }
        csv << "matrix_name,n,nnz,nnz_per_row,precond_setup_ms,solve_ms,iterations,converged,final_residual\n";
        char buf[96];
        for (const Row& r : rows) {
            std::snprintf(buf, sizeof buf, "%.2f,%.2f,%.2f", (double)r.nnz / (double)r.n, r.setup_ms, r.solve_ms);
            csv << r.name << "," << r.n << "," << r.nnz << "," << buf << "," << r.iterations << ","
                << (r.converged ? "true" : "false") << ",";
            std::snprintf(buf, sizeof buf, "%.17g", r.final_residual);
            csv << buf << "\n";
        }
    }
    return 0;
}

int cmd_partition(const std::string& matrix_path, index_t s, const std::string& out_path) {  // :349-363
    const SparseMatrix a = read_matrix(matrix_path);
    const WeightedGraph g = graph_from_matrix(a);
    Partition p = partition_graph(g, s, 0.1);
    measure_block_nnz(p, a);
    const double cut = cut_weight(g, p);
    std::ofstream out(out_path);
    if (!out) throw std::runtime_error("cannot open output file: " + out_path);
    export_partition(out, p);
    std::printf("blocks=%lld cut_weight=%.6g nnz_imbalance=%.4f\n", (long long)s, cut, p.imbalance);
    return 0;
}

void usage() {
    std::fprintf(stderr,
                 "usage: hpbj_cli solve --matrix A.mtx [options] | bench --specs S.json [--repetitions K] "
                 "[--out T.csv] | partition --matrix A.mtx --blocks S --out P.txt\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 1;
    }
    const std::string cmd = argv[1];
    std::map<std::string, std::string> opt;
    std::map<std::string, bool> flag;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--absolute-tol" || a == "--ritz") {
            flag[a] = true;
        } else if (a.rfind("--", 0) == 0 && i + 1 < argc) {
            opt[a] = argv[++i];
        } else {
            std::fprintf(stderr, "error: unexpected argument '%s'\n", a.c_str());
            usage();
            return 1;
        }
    }
    auto has = [&](const char* k) { return opt.count(k) > 0; };
    try {
        if (cmd == "solve") {
            RunSpec spec;
            if (!has("--matrix")) {
                std::fprintf(stderr, "error: --matrix is required\n");
                return 1;
            }
            spec.matrix_path = opt["--matrix"];
            if (has("--rhs")) spec.rhs_mode = opt["--rhs"];
            if (has("--precond")) spec.precond = opt["--precond"];
            if (has("--blocks")) spec.blocks = std::stoll(opt["--blocks"]);
            if (has("--restart")) spec.restart_m = std::stoll(opt["--restart"]);
            if (has("--tol")) spec.tol = std::stod(opt["--tol"]);
            if (has("--max-restarts")) spec.max_restarts = std::stoll(opt["--max-restarts"]);
            if (has("--precision")) spec.precision = opt["--precision"];
            if (has("--eps-pivot")) spec.eps_pivot = std::stod(opt["--eps-pivot"]);
            if (has("--neumann-order")) spec.neumann_order = std::stoi(opt["--neumann-order"]);
            if (has("--partition-file")) spec.partition_file = opt["--partition-file"];
            if (has("--report")) spec.report_path = opt["--report"];
            if (has("--history")) spec.history_path = opt["--history"];
            spec.absolute_tol = flag["--absolute-tol"];
            spec.ritz = flag["--ritz"];
            const std::string bad = check_spec(spec, has("--blocks"), has("--partition-file"), has("--neumann-order"),
                                               has("--eps-pivot"));
            if (!bad.empty()) {
                std::cerr << "error: " << bad << "\n";
                return 1;
            }
            const RunResult r = run_spec(spec);
            if (!spec.report_path.empty()) {
                std::ofstream out(spec.report_path);
                if (!out) throw std::runtime_error("cannot open report file: " + spec.report_path);
                out << report_json(spec, r);
            }
            if (!spec.history_path.empty()) write_history_csv(spec.history_path, r.report);
            print_summary(r);
            return r.report.converged ? 0 : 2;
        }
        if (cmd == "bench") {
            if (!has("--specs")) {
                std::fprintf(stderr, "error: --specs is required\n");
                return 1;
            }
            const int reps = has("--repetitions") ? std::stoi(opt["--repetitions"]) : 1;
            if (reps < 1) {
                std::fprintf(stderr, "error: --repetitions must be positive\n");
                return 1;
            }
            return cmd_bench(opt["--specs"], reps, has("--out") ? opt["--out"] : "");
        }
        if (cmd == "partition") {
            if (!has("--matrix") || !has("--blocks") || !has("--out")) {
                std::fprintf(stderr, "error: --matrix, --blocks and --out are required\n");
                return 1;
            }
            const index_t s = std::stoll(opt["--blocks"]);
            if (s < 1) {
                std::cerr << "error: --blocks must be >= 1\n";
                return 1;
            }
            return cmd_partition(opt["--matrix"], s, opt["--out"]);
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    usage();
    return 1;
}
