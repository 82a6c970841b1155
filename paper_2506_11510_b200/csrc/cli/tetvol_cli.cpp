// tetvol_b200: the reference CLI (cli.cpp) over the B200 library — the same
// subcommands (gen / build / render / compare / validate / stats), options,
// config-file format, JSON reports (schema 1, keys sorted as nlohmann::json
// prints them) and exit codes (0 ok, 1 failure, 2 usage or config error), with
// every compute step on the GPU through the C ABI (include/tetvol_b200.h).
//
// CLI11 and nlohmann::json are not available here; a small option parser and
// JSON writer/reader below stand in for them. Deviations from CLI11: help text
// layout and parse-error wording (the exit code, 2, is the same).
#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tetvol_b200.h"

namespace {

// ------------------------------------------------------------------ errors ---
struct CliError : std::runtime_error {
    int code;  // tv_status
    CliError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(int rc) {
    if (rc) throw CliError(rc, tv_last_error());
}
[[noreturn]] void config_error(const std::string& m) { throw CliError(TV_ERR_CONFIG, m); }

// -------------------------------------------------------------------- json ---
// A JSON value printed like nlohmann::json::dump(2): object keys sorted,
// two-space indent, doubles in shortest round-trip form with ".0" on integral
// values, non-finite doubles as null.
struct Json {
    enum Kind { Null, Bool, Int, UInt, Double, String, Array, Object } kind = Null;
    bool b = false;
    long long i = 0;
    unsigned long long u = 0;
    double d = 0;
    std::string s;
    std::vector<Json> a;
    std::map<std::string, Json> o;

    Json() = default;
    Json(std::nullptr_t) {}
    Json(bool v) : kind(Bool), b(v) {}
    Json(int v) : kind(Int), i(v) {}
    Json(long long v) : kind(Int), i(v) {}
    Json(unsigned v) : kind(UInt), u(v) {}
    Json(unsigned long v) : kind(UInt), u(v) {}
    Json(unsigned long long v) : kind(UInt), u(v) {}
    Json(double v) : kind(Double), d(v) {}
    Json(const char* v) : kind(String), s(v) {}
    Json(const std::string& v) : kind(String), s(v) {}
    static Json array(std::vector<Json> v) {
        Json j;
        j.kind = Array;
        j.a = std::move(v);
        return j;
    }
    static Json object() {
        Json j;
        j.kind = Object;
        return j;
    }
    Json& operator[](const std::string& k) {
        kind = Object;
        return o[k];
    }
    bool contains(const std::string& k) const { return kind == Object && o.count(k); }
    bool is_number() const { return kind == Int || kind == UInt || kind == Double; }
    double number() const { return kind == Int ? static_cast<double>(i) : kind == UInt ? static_cast<double>(u) : d; }
};

std::string fmt_double(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".en") == std::string::npos) s += ".0";
    return s;
}

void escape(std::ostream& out, const std::string& s) {
    out << '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out << "\\\""; break;
            case '\\': out << "\\\\"; break;
            case '\n': out << "\\n"; break;
            case '\r': out << "\\r"; break;
            case '\t': out << "\\t"; break;
            case '\b': out << "\\b"; break;
            case '\f': out << "\\f"; break;
            default:
                if (c < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", c);
                    out << b;
                } else {
                    out << c;
                }
        }
    }
    out << '"';
}

void dump(std::ostream& out, const Json& j, int indent) {
    const std::string pad(indent + 2, ' '), end(indent, ' ');
    switch (j.kind) {
        case Json::Null: out << "null"; break;
        case Json::Bool: out << (j.b ? "true" : "false"); break;
        case Json::Int: out << j.i; break;
        case Json::UInt: out << j.u; break;
        case Json::Double: out << fmt_double(j.d); break;
        case Json::String: escape(out, j.s); break;
        case Json::Array:
            if (j.a.empty()) {
                out << "[]";
                break;
            }
            out << "[\n";
            for (size_t k = 0; k < j.a.size(); ++k) {
                out << pad;
                dump(out, j.a[k], indent + 2);
                out << (k + 1 < j.a.size() ? ",\n" : "\n");
            }
            out << end << "]";
            break;
        case Json::Object:
            if (j.o.empty()) {
                out << "{}";
                break;
            }
            out << "{\n";
            for (auto it = j.o.begin(); it != j.o.end(); ++it) {
                out << pad;
                escape(out, it->first);
                out << ": ";
                dump(out, it->second, indent + 2);
                out << (std::next(it) != j.o.end() ? ",\n" : "\n");
            }
            out << end << "}";
            break;
    }
}

// minimal reader for the stats files compare consumes
struct JsonReader {
    const std::string& t;
    size_t p = 0;
    explicit JsonReader(const std::string& s) : t(s) {}
    [[noreturn]] void bad(const std::string& what) {
        throw std::runtime_error("parse error at byte " + std::to_string(p) + ": " + what);
    }
    void ws() {
        while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p]))) ++p;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (t.compare(p, n, w) == 0) {
            p += n;
            return true;
        }
        return false;
    }
    std::string str() {
        if (t[p] != '"') bad("expected string");
        ++p;
        std::string s;
        while (p < t.size() && t[p] != '"') {
            if (t[p] == '\\' && p + 1 < t.size()) {
                const char e = t[++p];
                s.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e);
                if (e == 'u') p += 4, s.back() = '?';
            } else {
                s.push_back(t[p]);
            }
            ++p;
        }
        if (p >= t.size()) bad("unterminated string");
        ++p;
        return s;
    }
    Json value() {
        ws();
        if (p >= t.size()) bad("unexpected end of input");
        const char c = t[p];
        if (c == '{') {
            ++p;
            Json j = Json::object();
            ws();
            if (p < t.size() && t[p] == '}') return ++p, j;
            for (;;) {
                ws();
                std::string k = str();
                ws();
                if (p >= t.size() || t[p] != ':') bad("expected ':'");
                ++p;
                j.o[k] = value();
                ws();
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == '}') return ++p, j;
                bad("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++p;
            Json j = Json::array({});
            ws();
            if (p < t.size() && t[p] == ']') return ++p, j;
            for (;;) {
                j.a.push_back(value());
                ws();
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == ']') return ++p, j;
                bad("expected ',' or ']'");
            }
        }
        if (c == '"') return Json(str());
        if (lit("true")) return Json(true);
        if (lit("false")) return Json(false);
        if (lit("null")) return Json();
        const size_t b = p;
        while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || std::strchr("+-.eE", t[p]))) ++p;
        if (b == p) bad("unexpected character");
        return Json(std::stod(t.substr(b, p - b)));
    }
};

void emit(const Json& j, const std::string& stats_path) {
    dump(std::cout, j, 0);
    std::cout << "\n";
    if (!stats_path.empty()) {
        std::ofstream f(stats_path);
        if (!f) throw CliError(TV_ERR_IO, "cannot open '" + stats_path + "' for writing");
        dump(f, j, 0);
        f << "\n";
    }
}

Json read_json_file(const std::string& path) {  // cli.cpp:296-306
    std::ifstream f(path);
    if (!f) throw CliError(TV_ERR_IO, "cannot open '" + path + "'");
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string text = ss.str();
    try {
        JsonReader r(text);
        Json j = r.value();
        r.ws();
        if (r.p != text.size()) r.bad("trailing characters");
        return j;
    } catch (const std::exception& e) {
        throw CliError(TV_ERR_FORMAT, path + ": " + e.what());
    }
}

double jnum(const Json& j, const char* key, const std::string& path) {  // cli.cpp:308-312
    if (!j.contains(key) || !j.o.at(key).is_number())
        throw CliError(TV_ERR_FORMAT, path + ": missing numeric field '" + std::string(key) + "'");
    return j.o.at(key).number();
}

// ---------------------------------------------------------- value parsing ---
// cli.cpp:34-117
std::string trim(const std::string& s) {
    const size_t b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return "";
    const size_t e = s.find_last_not_of(" \t\r\n");
    return s.substr(b, e - b + 1);
}

std::vector<std::string> split_fields(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == ',' || c == ' ' || c == '\t') {
            if (!cur.empty()) out.push_back(cur), cur.clear();
        } else {
            cur.push_back(c);
        }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}

double parse_double(const std::string& s, const std::string& what) {
    try {
        size_t pos = 0;
        const double v = std::stod(s, &pos);
        if (pos != s.size()) throw std::invalid_argument("trailing garbage");
        return v;
    } catch (const std::exception&) {
        config_error(what + ": not a number: '" + s + "'");
    }
}

long long parse_int(const std::string& s, const std::string& what) {
    try {
        size_t pos = 0;
        const long long v = std::stoll(s, &pos);
        if (pos != s.size()) throw std::invalid_argument("trailing garbage");
        return v;
    } catch (const std::exception&) {
        config_error(what + ": not an integer: '" + s + "'");
    }
}

uint64_t parse_u64(const std::string& s, const std::string& what) {
    try {
        size_t pos = 0;
        const unsigned long long v = std::stoull(s, &pos);
        if (pos != s.size()) throw std::invalid_argument("trailing garbage");
        return v;
    } catch (const std::exception&) {
        config_error(what + ": not an unsigned integer: '" + s + "'");
    }
}

bool parse_bool(const std::string& s, const std::string& what) {
    if (s == "true" || s == "1" || s == "yes" || s == "on") return true;
    if (s == "false" || s == "0" || s == "no" || s == "off") return false;
    config_error(what + ": not a boolean: '" + s + "'");
}

struct V3 {
    double x = 0, y = 0, z = 0;
};

V3 parse_vec3(const std::string& s, const std::string& what) {
    auto f = split_fields(s);
    if (f.size() != 3) config_error(what + ": expected 3 components, got '" + s + "'");
    return {parse_double(f[0], what), parse_double(f[1], what), parse_double(f[2], what)};
}

std::array<int, 3> parse_dims(const std::string& s) {
    std::string norm = s;
    std::replace(norm.begin(), norm.end(), 'x', ',');
    std::replace(norm.begin(), norm.end(), 'X', ',');
    auto f = split_fields(norm);
    if (f.size() == 1) {
        const int n = static_cast<int>(parse_int(f[0], "dims"));
        return {n, n, n};
    }
    if (f.size() == 3)
        return {static_cast<int>(parse_int(f[0], "dims")), static_cast<int>(parse_int(f[1], "dims")),
                static_cast<int>(parse_int(f[2], "dims"))};
    config_error("dims: expected N or NX,NY,NZ, got '" + s + "'");
}

// ---------------------------------------------------------------- settings ---
// cli.cpp:119-287: defaults <- config file <- command-line flags
struct CameraSettings {
    V3 position{0.5, 0.5, -2.0};
    std::optional<V3> look_at, forward;
    V3 up{0.0, 1.0, 0.0};
    double vfov = 45.0;
    int width = 256, height = 256;

    tv_camera make() const {
        if (look_at && forward) config_error("camera: set look_at or forward, not both");
        V3 f;
        if (forward) {
            f = *forward;
        } else {
            const V3 t = look_at ? *look_at : V3{0.5, 0.5, 0.5};
            f = {t.x - position.x, t.y - position.y, t.z - position.z};
        }
        tv_camera c{};
        c.position[0] = position.x, c.position[1] = position.y, c.position[2] = position.z;
        c.forward[0] = f.x, c.forward[1] = f.y, c.forward[2] = f.z;
        c.up[0] = up.x, c.up[1] = up.y, c.up[2] = up.z;
        c.vfov_degrees = vfov, c.width = width, c.height = height, c.basis_final = 0;
        check(tv_check_camera(&c));  // PinholeCamera's constructor throws CameraError here
        return c;
    }
};

struct Settings {
    CameraSettings camera;
    tv_build_config build{0.1, 24, 0, 1.0, 1.0};                                   // builder.hpp:21-29
    tv_render_config render{32, 64, 0, 0.0, 0.8, {1.0, 1.0, 1.0}, 1.0, 1.0, 2.2};  // tracer.hpp:16-28
    int threads = 0;
};

void apply_setting(Settings& s, const std::string& section, const std::string& key, const std::string& value) {
    const std::string what = section + "." + key;
    if (section == "camera") {
        if (key == "position") s.camera.position = parse_vec3(value, what);
        else if (key == "look_at") s.camera.look_at = parse_vec3(value, what);
        else if (key == "forward") s.camera.forward = parse_vec3(value, what);
        else if (key == "up") s.camera.up = parse_vec3(value, what);
        else if (key == "vfov") s.camera.vfov = parse_double(value, what);
        else if (key == "width") s.camera.width = static_cast<int>(parse_int(value, what));
        else if (key == "height") s.camera.height = static_cast<int>(parse_int(value, what));
        else config_error("config: unknown key '" + what + "'");
    } else if (section == "build") {
        if (key == "threshold") s.build.variation_threshold = parse_double(value, what);
        else if (key == "max_level") s.build.max_level = static_cast<int>(parse_int(value, what));
        else if (key == "use_camera") s.build.use_camera = parse_bool(value, what);
        else if (key == "pixel_threshold") s.build.pixel_threshold = parse_double(value, what);
        else if (key == "density_scale") s.build.density_scale = parse_double(value, what);
        else config_error("config: unknown key '" + what + "'");
    } else if (section == "render") {
        if (key == "spp") s.render.spp = static_cast<int>(parse_int(value, what));
        else if (key == "max_bounces") s.render.max_bounces = static_cast<int>(parse_int(value, what));
        else if (key == "seed") s.render.seed = parse_u64(value, what);
        else if (key == "g") s.render.hg_g = parse_double(value, what);
        else if (key == "albedo") s.render.default_albedo = parse_double(value, what);
        else if (key == "environment") {
            const V3 e = parse_vec3(value, what);
            s.render.environment[0] = e.x, s.render.environment[1] = e.y, s.render.environment[2] = e.z;
        } else if (key == "emission_scale") s.render.emission_scale = parse_double(value, what);
        else if (key == "exposure") s.render.exposure = parse_double(value, what);
        else if (key == "gamma") s.render.gamma = parse_double(value, what);
        else if (key == "threads") s.threads = static_cast<int>(parse_int(value, what));
        else config_error("config: unknown key '" + what + "'");
    } else {
        config_error("config: unknown section '[" + section + "]'");
    }
}

void load_config_file(const std::string& path, Settings& s) {
    std::ifstream f(path);
    if (!f) config_error("config: cannot open '" + path + "'");
    std::string line, section;
    int lineno = 0;
    while (std::getline(f, line)) {
        ++lineno;
        const size_t hash = line.find('#');
        if (hash != std::string::npos) line.erase(hash);
        line = trim(line);
        if (line.empty()) continue;
        if (line.front() == '[') {
            if (line.back() != ']') config_error("config: bad section header at line " + std::to_string(lineno));
            section = trim(line.substr(1, line.size() - 2));
            continue;
        }
        const size_t eq = line.find('=');
        if (eq == std::string::npos) config_error("config: expected key = value at line " + std::to_string(lineno));
        const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
        if (key.empty() || value.empty()) config_error("config: empty key or value at line " + std::to_string(lineno));
        if (section.empty()) config_error("config: key '" + key + "' before any [section]");
        apply_setting(s, section, key, value);
    }
}

// ------------------------------------------------------------- arg parsing ---
// A CLI11 stand-in: "--name value", "--name=value", flags, required options,
// mutually exclusive options; all values are kept as strings and converted the
// way CLI11 converts them (integers, doubles, u64).
struct Opt {
    std::string name, help;
    bool flag = false, required = false;
    std::vector<std::string> values;
    bool given() const { return !values.empty(); }
    const std::string& value() const { return values.back(); }
};

struct Command {
    std::string name, help;
    std::vector<Opt> opts;
    std::vector<std::pair<std::string, std::string>> excludes, needs;  // (a, b)
    Opt& add(const std::string& n, const std::string& h, bool flag = false, bool req = false) {
        opts.push_back(Opt{n, h, flag, req, {}});
        return opts.back();
    }
    Opt* find(const std::string& n) {
        for (auto& o : opts)
            if (o.name == n) return &o;
        return nullptr;
    }
    const Opt& get(const std::string& n) const {
        for (auto& o : opts)
            if (o.name == n) return o;
        throw std::logic_error("no option " + n);
    }
    bool has(const std::string& n) const { return get(n).given(); }
    std::string str(const std::string& n, const std::string& def = "") const { return has(n) ? get(n).value() : def; }
    void usage(std::ostream& out) const {
        out << "Usage: tetvol_b200 " << name << " [OPTIONS]\n\n" << help << "\n\nOptions:\n";
        for (auto& o : opts)
            out << "  " << o.name << (o.flag ? "" : " VALUE") << (o.required ? " REQUIRED" : "") << "\n      "
                << o.help << "\n";
    }
    void parse(const std::vector<std::string>& args) {
        for (size_t k = 0; k < args.size(); ++k) {
            std::string a = args[k], val;
            bool has_val = false;
            const size_t eq = a.find('=');
            if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = a.substr(eq + 1), a = a.substr(0, eq), has_val = true;
            }
            Opt* o = find(a);
            if (!o) throw UsageError("The following argument was not expected: " + args[k]);
            if (o->flag) {
                if (has_val) throw UsageError(a + ": flag does not take a value");
                o->values.push_back("1");
                continue;
            }
            if (!has_val) {
                if (k + 1 >= args.size()) throw UsageError(a + ": 1 required VALUE missing");
                val = args[++k];
            }
            o->values.push_back(val);
        }
        for (auto& o : opts)
            if (o.required && !o.given()) throw UsageError(o.name + " is required");
        for (auto& [x, y] : excludes)
            if (has(x) && has(y)) throw UsageError(x + " excludes " + y);
        for (auto& [x, y] : needs)
            if (has(x) && !has(y)) throw UsageError(x + " requires " + y);
    }
};

template <class T>
T conv(const Opt& o);
template <>
double conv<double>(const Opt& o) {
    try {
        size_t pos = 0;
        const double v = std::stod(o.value(), &pos);
        if (pos == o.value().size()) return v;
    } catch (...) {
    }
    throw UsageError(o.name + ": Value " + o.value() + " could not be converted");
}
template <>
int conv<int>(const Opt& o) {
    try {
        size_t pos = 0;
        const long long v = std::stoll(o.value(), &pos);
        if (pos == o.value().size() && v >= INT32_MIN && v <= INT32_MAX) return static_cast<int>(v);
    } catch (...) {
    }
    throw UsageError(o.name + ": Value " + o.value() + " could not be converted");
}
template <>
uint64_t conv<uint64_t>(const Opt& o) {
    try {
        size_t pos = 0;
        if (!o.value().empty() && o.value()[0] != '-') {
            const unsigned long long v = std::stoull(o.value(), &pos);
            if (pos == o.value().size()) return v;
        }
    } catch (...) {
    }
    throw UsageError(o.name + ": Value " + o.value() + " could not be converted");
}

void add_camera_options(Command& c) {  // cli.cpp:229-237
    c.add("--position", "camera position 'x,y,z'");
    c.add("--look-at", "camera target 'x,y,z'");
    c.add("--forward", "view direction 'x,y,z' (alternative to --look-at)");
    c.add("--up", "up vector 'x,y,z'");
    c.add("--vfov", "vertical field of view, degrees");
    c.add("--width", "image width in pixels");
    c.add("--height", "image height in pixels");
}

void add_build_options(Command& c) {  // cli.cpp:239-246
    c.add("--threshold", "refine while (max-min)/mean exceeds this");
    c.add("--max-level", "maximum bisection depth");
    c.add("--use-camera", "skip refinement outside the view frustum", true);
    c.add("--no-use-camera", "force view-independent refinement", true);
    c.add("--pixel-threshold", "minimum projected size worth refining, pixels");
    c.add("--density-scale", "extinction = scale * density");
}

void add_render_options(Command& c) {  // cli.cpp:248-259
    c.add("--spp", "samples per pixel");
    c.add("--max-bounces", "path length cap");
    c.add("--seed", "RNG seed");
    c.add("--g", "Henyey-Greenstein anisotropy in (-1,1)");
    c.add("--albedo", "scattering albedo for cells without their own");
    c.add("--environment", "escape radiance 'r,g,b'");
    c.add("--emission-scale", "emission strength multiplier");
    c.add("--exposure", "linear exposure for 8-bit output");
    c.add("--gamma", "gamma for 8-bit output");
    c.add("--threads", "worker threads (0 = all cores); accepted, the GPU does the work");
}

// cli.cpp:261-287 (only options the user passed override the config file)
Settings resolve_settings(const Command& c) {
    Settings s;
    if (c.has("--config")) load_config_file(c.str("--config"), s);
    auto has = [&](const char* n) {
        for (auto& o : c.opts)
            if (o.name == n) return o.given();
        return false;
    };
    auto get = [&](const char* n) -> const Opt& { return c.get(n); };
    if (has("--position")) s.camera.position = parse_vec3(get("--position").value(), "--position");
    if (has("--look-at")) s.camera.look_at = parse_vec3(get("--look-at").value(), "--look-at");
    if (has("--forward")) s.camera.forward = parse_vec3(get("--forward").value(), "--forward");
    if (has("--up")) s.camera.up = parse_vec3(get("--up").value(), "--up");
    if (has("--vfov")) s.camera.vfov = conv<double>(get("--vfov"));
    if (has("--width")) s.camera.width = conv<int>(get("--width"));
    if (has("--height")) s.camera.height = conv<int>(get("--height"));
    if (has("--threshold")) s.build.variation_threshold = conv<double>(get("--threshold"));
    if (has("--max-level")) s.build.max_level = conv<int>(get("--max-level"));
    if (has("--use-camera") && has("--no-use-camera")) config_error("--use-camera conflicts with --no-use-camera");
    if (has("--use-camera")) s.build.use_camera = 1;
    if (has("--no-use-camera")) s.build.use_camera = 0;
    if (has("--pixel-threshold")) s.build.pixel_threshold = conv<double>(get("--pixel-threshold"));
    if (has("--density-scale")) s.build.density_scale = conv<double>(get("--density-scale"));
    if (has("--spp")) s.render.spp = conv<int>(get("--spp"));
    if (has("--max-bounces")) s.render.max_bounces = conv<int>(get("--max-bounces"));
    if (has("--seed")) s.render.seed = conv<uint64_t>(get("--seed"));
    if (has("--g")) s.render.hg_g = conv<double>(get("--g"));
    if (has("--albedo")) s.render.default_albedo = conv<double>(get("--albedo"));
    if (has("--environment")) {
        const V3 e = parse_vec3(get("--environment").value(), "--environment");
        s.render.environment[0] = e.x, s.render.environment[1] = e.y, s.render.environment[2] = e.z;
    }
    if (has("--emission-scale")) s.render.emission_scale = conv<double>(get("--emission-scale"));
    if (has("--exposure")) s.render.exposure = conv<double>(get("--exposure"));
    if (has("--gamma")) s.render.gamma = conv<double>(get("--gamma"));
    if (has("--threads")) s.threads = conv<int>(get("--threads"));
    return s;
}

// ------------------------------------------------------------------ handles ---
struct Grid {
    tv_grid* h = nullptr;
    ~Grid() { tv_grid_free(h); }
};
struct Volume {
    tv_volume* h = nullptr;
    ~Volume() { tv_volume_free(h); }
};

std::vector<std::string> channel_names(const tv_volume* v) {
    int32_t n = 0;
    check(tv_volume_get_info(v, nullptr, &n));
    std::vector<std::string> out;
    char buf[256];
    for (int32_t i = 0; i < n; ++i) {
        check(tv_volume_channel_name(v, i, buf, sizeof(buf)));
        out.emplace_back(buf);
    }
    return out;
}

Json str_array(const std::vector<std::string>& v) {
    std::vector<Json> a;
    for (auto& s : v) a.emplace_back(s);
    return Json::array(a);
}

// --------------------------------------------------------------------- gen ---
int cmd_gen(const Command& c) {  // cli.cpp:349-391
    const std::string kind = c.str("--kind"), out = c.str("--out");
    const auto dims = parse_dims(c.str("--dims", "64"));
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || dims[0] > 4096 || dims[1] > 4096 || dims[2] > 4096)
        config_error("dims out of range [1, 4096]");
    static const std::map<std::string, int> kinds{{"constant", 0}, {"ramp", 1}, {"blob", 2},
                                                  {"step", 3},     {"noise", 4}, {"cloud", 5}};
    auto it = kinds.find(kind);
    // the reference's message; 'cloud' is accepted as an extension
    if (it == kinds.end()) config_error("unknown kind '" + kind + "' (constant|ramp|blob|step|noise)");
    const double value = c.has("--value") ? conv<double>(c.get("--value")) : 1.0;
    Volume v;
    check(tv_volume_create(dims[0], dims[1], dims[2], 0, &v.h));
    check(tv_volume_generate(v.h, it->second, value));
    if (c.has("--with-temperature")) check(tv_volume_add_temperature(v.h));
    if (c.has("--with-albedo")) check(tv_volume_add_albedo(v.h, conv<double>(c.get("--with-albedo"))));
    check(tv_volume_save(v.h, out.c_str()));
    Json j = Json::object();
    j["schema"] = 1;
    j["command"] = "gen";
    j["kind"] = kind;
    j["dims"] = Json::array({dims[0], dims[1], dims[2]});
    j["channels"] = str_array(channel_names(v.h));
    j["out"] = out;
    emit(j, c.str("--stats-out"));
    return 0;
}

// ------------------------------------------------------------------- build ---
int cmd_build(const Command& c) {  // cli.cpp:395-423
    Settings s = resolve_settings(c);
    Volume v;
    check(tv_volume_load(c.str("--volume").c_str(), 0, &v.h));
    std::optional<tv_camera> cam;
    if (s.build.use_camera) cam = s.camera.make();
    Grid g;
    tv_build_stats bs{};
    check(tv_build_volume(v.h, &s.build, cam ? &*cam : nullptr, &g.h, &bs));
    tv_validation_report vr{};
    check(tv_grid_validate(g.h, &vr));
    if (!vr.ok) {
        std::cerr << "built grid failed validation: " << vr.first_violation << "\n";
        return 1;
    }
    const std::string out = c.str("--out");
    check(tv_grid_save(g.h, out.c_str()));
    tv_grid_info gi{};
    check(tv_grid_get_info(g.h, &gi));
    Json j = Json::object();
    j["schema"] = 1;
    j["command"] = "build";
    j["leafCount"] = static_cast<unsigned long long>(bs.leaf_count);
    j["maxDepthReached"] = bs.max_depth;
    j["buildSeconds"] = bs.seconds;
    j["criterionSplits"] = static_cast<unsigned long long>(bs.criterion_splits);
    j["propagationSplits"] = static_cast<unsigned long long>(bs.propagation_splits);
    j["tetCount"] = static_cast<unsigned long long>(gi.n_tets);
    j["vertexCount"] = static_cast<unsigned long long>(gi.n_vertices);
    j["out"] = out;
    emit(j, c.str("--stats-out"));
    return 0;
}

// ------------------------------------------------------------------ render ---
// image.cpp:13-31
void write_ppm(const std::string& path, int w, int h, const std::vector<double>& sum,
               const std::vector<uint32_t>& counts, double exposure, double gamma) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw CliError(TV_ERR_IMAGE, "cannot open for writing: " + path);
    f << "P6\n" << w << " " << h << "\n255\n";
    std::vector<unsigned char> row(static_cast<size_t>(w) * 3);
    const double inv_gamma = 1.0 / gamma;
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const size_t p = static_cast<size_t>(y) * w + x;
            const uint32_t n = counts[p];
            for (int k = 0; k < 3; ++k) {
                const double m = n == 0 ? 0.0 : sum[3 * p + k] / n;  // ImageAccumulator::mean
                const double e = std::pow(std::clamp(m * exposure, 0.0, 1.0), inv_gamma);
                row[static_cast<size_t>(x) * 3 + k] = static_cast<unsigned char>(e * 255.0 + 0.5);
            }
        }
        f.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size()));
    }
    if (!f) throw CliError(TV_ERR_IMAGE, "write failed: " + path);
}

int cmd_render(const Command& c) {  // cli.cpp:427-482
    if (!c.has("--grid") && !c.has("--volume")) config_error("render needs --grid or --volume");
    Settings s = resolve_settings(c);
    const tv_camera cam = s.camera.make();
    check(tv_check_render_config(&s.render));  // s.render.validate() (cli.cpp:430)
    const int w = cam.width, h = cam.height;
    tv_framebuffer fb{};
    std::vector<double> sum, sum_sq;
    std::vector<uint32_t> counts;
    tv_render_stats st{};
    std::string mode;
    unsigned long long cell_count = 0;
    if (w >= 1 && h >= 1) {
        sum.resize(static_cast<size_t>(w) * h * 3), sum_sq.resize(sum.size()), counts.resize(static_cast<size_t>(w) * h);
        fb.sum = sum.data(), fb.sum_sq = sum_sq.data(), fb.sample_counts = counts.data();
    }
    if (c.has("--reference")) {
        Volume v;
        check(tv_volume_load(c.str("--volume").c_str(), 0, &v.h));
        float* dens = nullptr;
        check(tv_volume_channel_dev(v.h, "density", &dens));
        int32_t dims[3];
        check(tv_volume_get_info(v.h, dims, nullptr));
        check(tv_render_regular_dev(dens, dims[0], dims[1], dims[2], s.build.density_scale, &cam, &s.render, 0, &fb,
                                    &st));
        mode = "reference";
        cell_count = static_cast<unsigned long long>(dims[0]) * dims[1] * dims[2];
    } else {
        Grid g;
        if (c.has("--grid")) {
            check(tv_grid_load(c.str("--grid").c_str(), 0, &g.h));
        } else {
            Volume v;
            check(tv_volume_load(c.str("--volume").c_str(), 0, &v.h));
            std::optional<tv_camera> bcam;
            if (s.build.use_camera) bcam = s.camera.make();
            std::cerr << "building adaptive grid from '" << c.str("--volume") << "'\n";
            tv_build_stats bs{};
            check(tv_build_volume(v.h, &s.build, bcam ? &*bcam : nullptr, &g.h, &bs));
        }
        check(tv_render(g.h, &cam, &s.render, &fb, &st));
        mode = "tet";
        tv_grid_info gi{};
        check(tv_grid_get_info(g.h, &gi));
        cell_count = gi.n_leaves;
    }
    if (c.has("--ppm")) write_ppm(c.str("--ppm"), w, h, sum, counts, s.render.exposure, s.render.gamma);
    if (c.has("--pfm")) check(tv_image_write_pfm(c.str("--pfm").c_str(), &fb, w, h, 0, 0, 0));
    if (c.has("--var-pfm")) check(tv_image_write_pfm(c.str("--var-pfm").c_str(), &fb, w, h, 1, 0, 0));
    Json j = Json::object();
    j["schema"] = 1;
    j["command"] = "render";
    j["mode"] = mode;
    j["width"] = w;
    j["height"] = h;
    j["spp"] = s.render.spp;
    j["seed"] = static_cast<unsigned long long>(s.render.seed);
    j["cellCount"] = cell_count;
    j["paths"] = static_cast<unsigned long long>(st.paths_traced);
    j["cellsVisited"] = static_cast<unsigned long long>(st.cells_visited);
    j["meanCellsPerPath"] = st.paths_traced ? static_cast<double>(st.cells_visited) / static_cast<double>(st.paths_traced)
                                            : 0.0;
    j["degeneratePaths"] = static_cast<unsigned long long>(st.degenerate_paths);
    j["seconds"] = st.seconds;
    if (c.has("--ppm")) j["ppm"] = c.str("--ppm");
    if (c.has("--pfm")) j["pfm"] = c.str("--pfm");
    if (c.has("--var-pfm")) j["variancePfm"] = c.str("--var-pfm");
    emit(j, c.str("--stats-out"));
    return 0;
}

// ----------------------------------------------------------------- compare ---
struct Img {
    int w = 0, h = 0;
    std::vector<float> rgb;
};

Img read_pfm(const std::string& path) {
    Img im;
    check(tv_pfm_read(path.c_str(), &im.w, &im.h, nullptr));
    im.rgb.resize(static_cast<size_t>(im.w) * im.h * 3);
    check(tv_pfm_read(path.c_str(), &im.w, &im.h, im.rgb.data()));
    return im;
}

int cmd_compare(const Command& c) {  // cli.cpp:487-550
    const Img a = read_pfm(c.str("--image-a")), b = read_pfm(c.str("--image-b"));
    if (a.w != b.w || a.h != b.h)
        throw CliError(TV_ERR_FORMAT, "image dimensions differ: " + std::to_string(a.w) + "x" + std::to_string(a.h) +
                                          " vs " + std::to_string(b.w) + "x" + std::to_string(b.h));
    std::optional<Img> va, vb;
    if (c.has("--var-a") || c.has("--var-b")) {
        if (!c.has("--var-a") || !c.has("--var-b")) config_error("--var-a and --var-b must be given together");
        va = read_pfm(c.str("--var-a")), vb = read_pfm(c.str("--var-b"));
        if (va->w != a.w || va->h != a.h || vb->w != a.w || vb->h != a.h)
            throw CliError(TV_ERR_FORMAT, "variance image dimensions do not match the images");
    }
    tv_compare_stats cs{};
    check(tv_image_compare(a.rgb.data(), b.rgb.data(), va ? va->rgb.data() : nullptr, vb ? vb->rgb.data() : nullptr,
                           static_cast<uint64_t>(a.w) * a.h, 0, &cs));
    const std::string sa = c.str("--stats-a"), sb = c.str("--stats-b");
    const Json ja = read_json_file(sa), jb = read_json_file(sb);
    const double sec_a = jnum(ja, "seconds", sa), sec_b = jnum(jb, "seconds", sb);
    const double paths_a = jnum(ja, "paths", sa), paths_b = jnum(jb, "paths", sb);
    const double cells_a = jnum(ja, "cellsVisited", sa), cells_b = jnum(jb, "cellsVisited", sb);
    const double count_a = jnum(ja, "cellCount", sa), count_b = jnum(jb, "cellCount", sb);
    const double mean_a = paths_a > 0 ? cells_a / paths_a : 0.0, mean_b = paths_b > 0 ? cells_b / paths_b : 0.0;
    Json j = Json::object();
    j["schema"] = 1;
    j["command"] = "compare";
    j["width"] = a.w;
    j["height"] = a.h;
    j["rmse"] = cs.rmse;
    j["maxAbsDiff"] = cs.max_abs_diff;
    j["outlierFraction"] = va ? Json(cs.outlier_fraction) : Json();
    j["speedup"] = sec_a > 0 ? sec_b / sec_a : 0.0;
    j["cellsVisitedRatio"] = mean_a > 0 ? mean_b / mean_a : 0.0;
    j["cellCountRatio"] = count_a > 0 ? count_b / count_a : 0.0;
    emit(j, c.str("--stats-out"));
    return 0;
}

// ---------------------------------------------------------------- validate ---
int cmd_validate(const Command& c) {  // cli.cpp:560-604
    Grid g;
    check(tv_grid_load(c.str("--grid").c_str(), 0, &g.h));
    const int rays = c.has("--rays") ? conv<int>(c.get("--rays")) : 100;
    const uint64_t seed = c.has("--seed") ? conv<uint64_t>(c.get("--seed")) : 0;
    tv_validation_report vr{};
    check(tv_grid_validate(g.h, &vr));
    int32_t failures = 0, first = -1;
    if (vr.ok && rays > 0) {
        std::vector<tv_ray> r(rays);
        check(tv_validate_spot_rays(seed, rays, r.data()));
        check(tv_validate_rays(g.h, r.data(), rays, &failures, &first));
    }
    const bool ok = vr.ok && failures == 0;
    const std::string violation =
        !vr.ok ? std::string(vr.first_violation)
               : (failures ? "traversal mismatch vs brute-force oracle on spot-check ray " + std::to_string(first)
                           : std::string());
    Json j = Json::object();
    j["schema"] = 1;
    j["command"] = "validate";
    j["ok"] = ok;
    j["firstViolation"] = ok ? Json() : Json(violation);
    j["leafCount"] = static_cast<unsigned long long>(vr.leaf_count);
    j["interiorFaces"] = static_cast<unsigned long long>(vr.interior_faces);
    j["boundaryFaces"] = static_cast<unsigned long long>(vr.boundary_faces);
    j["rayChecks"] = vr.ok ? rays : 0;
    j["rayFailures"] = failures;
    emit(j, c.str("--stats-out"));
    if (ok)
        std::cerr << "grid OK: " << vr.leaf_count << " leaves, " << vr.interior_faces << " interior faces\n";
    else
        std::cerr << "grid INVALID: " << violation << "\n";
    return ok ? 0 : 1;
}

// ------------------------------------------------------------------- stats ---
int cmd_stats(const Command& c) {  // cli.cpp:608-677
    if (!c.has("--grid") && !c.has("--volume")) config_error("stats needs --grid or --volume");
    Json j = Json::object();
    j["schema"] = 1;
    j["command"] = "stats";
    if (c.has("--grid")) {
        Grid g;
        check(tv_grid_load(c.str("--grid").c_str(), 0, &g.h));
        tv_grid_info gi{};
        check(tv_grid_get_info(g.h, &gi));
        std::vector<tv_tet> tets(gi.n_tets);
        check(tv_grid_download(g.h, nullptr, tets.data(), nullptr));
        int max_level = 0;
        std::vector<unsigned long long> per_level;
        double min_d = 0.0, max_d = 0.0, sum_d = 0.0;
        bool first = true;
        for (const tv_tet& t : tets) {  // leaf_ids() order
            if (t.children[0] != TV_NO_TET) continue;
            max_level = std::max(max_level, static_cast<int>(t.level));
            if (per_level.size() <= t.level) per_level.resize(t.level + 1, 0);
            ++per_level[t.level];
            const double d = t.density;
            if (first) min_d = max_d = d, first = false;
            min_d = std::min(min_d, d);
            max_d = std::max(max_d, d);
            sum_d += d;
        }
        std::vector<Json> pl(per_level.begin(), per_level.end());
        j["kind"] = "grid";
        j["leafCount"] = static_cast<unsigned long long>(gi.n_leaves);
        j["tetCount"] = static_cast<unsigned long long>(gi.n_tets);
        j["vertexCount"] = static_cast<unsigned long long>(gi.n_vertices);
        j["maxLeafLevel"] = max_level;
        j["leavesPerLevel"] = Json::array(pl);
        Json d = Json::object();
        d["min"] = min_d;
        d["max"] = max_d;
        d["mean"] = gi.n_leaves ? sum_d / static_cast<double>(gi.n_leaves) : 0.0;
        j["density"] = d;
    } else {
        Volume v;
        check(tv_volume_load(c.str("--volume").c_str(), 0, &v.h));
        int32_t dims[3];
        check(tv_volume_get_info(v.h, dims, nullptr));
        j["kind"] = "volume";
        j["dims"] = Json::array({dims[0], dims[1], dims[2]});
        std::vector<Json> chans;
        std::vector<float> data(static_cast<size_t>(dims[0]) * dims[1] * dims[2]);
        for (const std::string& name : channel_names(v.h)) {
            check(tv_volume_download(v.h, name.c_str(), data.data()));
            double mn = 0.0, mx = 0.0, sum = 0.0;
            if (!data.empty()) {
                mn = mx = data[0];
                for (float x : data) {
                    mn = std::min(mn, static_cast<double>(x));
                    mx = std::max(mx, static_cast<double>(x));
                    sum += x;
                }
            }
            Json ch = Json::object();
            ch["name"] = name;
            ch["min"] = mn;
            ch["max"] = mx;
            ch["mean"] = data.empty() ? 0.0 : sum / static_cast<double>(data.size());
            chans.push_back(ch);
        }
        j["channels"] = Json::array(chans);
    }
    emit(j, c.str("--stats-out"));
    return 0;
}

// --------------------------------------------------------------------- main ---
std::vector<Command> commands() {
    std::vector<Command> cs;
    {
        Command c{"gen", "write a procedural test volume (.dvol)"};
        c.add("--kind", "constant|ramp|blob|step|noise (and cloud, SURVEY.md 8(d))", false, true);
        c.add("--dims", "N or NX,NY,NZ voxels");
        c.add("--out", "output .dvol path", false, true);
        c.add("--value", "density of the constant kind");
        c.add("--with-temperature", "add a temperature channel (= density)", true);
        c.add("--with-albedo", "add a constant albedo channel");
        c.add("--stats-out", "also write the JSON stats to this file");
        cs.push_back(c);
    }
    {
        Command c{"build", "build an adaptive tetrahedral grid (.tgrid) from a volume"};
        c.add("--volume", "input .dvol", false, true);
        c.add("--out", "output .tgrid path", false, true);
        c.add("--config", "config file ([camera]/[build]/[render] sections)");
        c.add("--stats-out", "also write the JSON stats to this file");
        add_build_options(c);
        add_camera_options(c);
        cs.push_back(c);
    }
    {
        Command c{"render", "path-trace a grid or a reference voxel volume"};
        c.add("--grid", "input .tgrid");
        c.add("--volume", "input .dvol");
        c.add("--reference", "render the voxel volume directly (needs --volume)", true);
        c.add("--config", "config file ([camera]/[build]/[render] sections)");
        c.add("--ppm", "8-bit tonemapped output path");
        c.add("--pfm", "linear float output path");
        c.add("--var-pfm", "per-pixel variance-of-mean output path");
        c.add("--stats-out", "also write the JSON stats to this file");
        add_render_options(c);
        add_build_options(c);
        add_camera_options(c);
        c.excludes = {{"--grid", "--volume"}};
        c.needs = {{"--reference", "--volume"}};
        cs.push_back(c);
    }
    {
        Command c{"compare", "compare two renders (grid render vs reference render)"};
        c.add("--image-a", "first linear image (.pfm), typically the grid render", false, true);
        c.add("--image-b", "second linear image (.pfm), typically the reference", false, true);
        c.add("--stats-a", "render stats JSON for image A", false, true);
        c.add("--stats-b", "render stats JSON for image B", false, true);
        c.add("--var-a", "variance image for A (enables the 3-sigma outlier test)");
        c.add("--var-b", "variance image for B");
        c.add("--stats-out", "also write the JSON report to this file");
        cs.push_back(c);
    }
    {
        Command c{"validate", "structural validation plus traversal spot checks"};
        c.add("--grid", "input .tgrid", false, true);
        c.add("--rays", "number of random spot-check rays");
        c.add("--seed", "spot-check RNG seed");
        c.add("--stats-out", "also write the JSON report to this file");
        cs.push_back(c);
    }
    {
        Command c{"stats", "summarize a grid or a volume file"};
        c.add("--grid", "input .tgrid");
        c.add("--volume", "input .dvol");
        c.add("--stats-out", "also write the JSON stats to this file");
        c.excludes = {{"--grid", "--volume"}};
        cs.push_back(c);
    }
    return cs;
}

void usage(std::ostream& out, const std::vector<Command>& cs) {
    out << "adaptive tetrahedral volume grids: build, render, compare (B200)\n"
           "Usage: tetvol_b200 SUBCOMMAND [OPTIONS]\n\nSubcommands:\n";
    for (auto& c : cs) out << "  " << c.name << "  " << c.help << "\n";
}

}  // namespace

// run() of cli.cpp:681-799: exit 0 ok, 1 runtime failure, 2 usage / config / camera error
int main(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    auto cs = commands();
    if (args.empty()) {
        usage(std::cerr, cs);
        std::cerr << "A subcommand is required\n";
        return 2;
    }
    if (args[0] == "-h" || args[0] == "--help") {
        usage(std::cout, cs);
        return 0;
    }
    auto it = std::find_if(cs.begin(), cs.end(), [&](const Command& c) { return c.name == args[0]; });
    if (it == cs.end()) {
        usage(std::cerr, cs);
        std::cerr << "The following argument was not expected: " << args[0] << "\n";
        return 2;
    }
    Command& c = *it;
    const std::vector<std::string> rest(args.begin() + 1, args.end());
    if (std::find(rest.begin(), rest.end(), "--help") != rest.end() ||
        std::find(rest.begin(), rest.end(), "-h") != rest.end()) {
        c.usage(std::cout);
        return 0;
    }
    try {
        c.parse(rest);
        if (c.name == "gen") return cmd_gen(c);
        if (c.name == "build") return cmd_build(c);
        if (c.name == "render") return cmd_render(c);
        if (c.name == "compare") return cmd_compare(c);
        if (c.name == "validate") return cmd_validate(c);
        return cmd_stats(c);
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 2;
    } catch (const CliError& e) {
        if (e.code == TV_ERR_CONFIG || e.code == TV_ERR_CAMERA) {
            std::cerr << "config error: " << e.what() << "\n";
            return 2;
        }
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
