// model.cu — the reference's on-disk contract feeding the hot path (SURVEY.md
// §8f row 2): the recipe JSON (schemas.cpp:240-298 parse_recipe_json) and the
// FQTA tensor archive (archive.cpp:123-192 decode_archive) are read on the host
// and turned into device layer handles, the way the CLI's load_recipes
// (flattenquant_cli.cpp:241-252) builds runnable LayerQuantConfigs; cmd_infer
// (flattenquant_cli.cpp:254-281) runs every "<layer>/<name>" input tensor of an
// archive through its layer and writes the outputs as an FQTA archive.
//
// Host-only code: a minimal JSON reader (objects, arrays, strings, numbers,
// literals; numbers parsed with strtod/strtoll as nlohmann/json does) and the
// FQTA reader/writer with the reference's validation and error texts.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <unordered_set>
#include <vector>

#include "fqg_internal.h"

namespace fqg {
namespace {

// ------------------------------------------------------------------ JSON
struct Json {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    std::string text;  // number literal or string value
    std::vector<Json> items;
    std::vector<std::pair<std::string, Json>> fields;

    const Json& at(const std::string& key) const {
        if (kind != Object) throw Error(FQG_ERR_INVALID, "recipe: expected an object for '" + key + "'");
        for (const auto& f : fields)
            if (f.first == key) return f.second;
        throw Error(FQG_ERR_INVALID, "recipe: missing key '" + key + "'");
    }
    double num() const {
        if (kind != Number) throw Error(FQG_ERR_INVALID, "recipe: expected a number");
        return std::strtod(text.c_str(), nullptr);
    }
    int64_t integer() const {
        if (kind != Number) throw Error(FQG_ERR_INVALID, "recipe: expected an integer");
        char* end = nullptr;
        errno = 0;
        const long long v = std::strtoll(text.c_str(), &end, 10);
        if (errno != 0 || end == nullptr || *end != '\0')
            throw Error(FQG_ERR_INVALID, "recipe: expected an integer, got " + text);
        return v;
    }
    const std::string& str() const {
        if (kind != String) throw Error(FQG_ERR_INVALID, "recipe: expected a string");
        return text;
    }
};

class JsonParser {
   public:
    explicit JsonParser(const std::string& s) : s_(s) {}
    Json parse() {
        Json v = value();
        ws();
        if (i_ != s_.size()) fail("trailing characters");
        return v;
    }

   private:
    [[noreturn]] void fail(const char* what) {
        throw Error(FQG_ERR_INVALID, std::string("recipe JSON: ") + what + " at offset " +
                                         std::to_string(i_));
    }
    void ws() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t'))
            ++i_;
    }
    Json value() {
        ws();
        if (i_ >= s_.size()) fail("unexpected end");
        const char c = s_[i_];
        Json v;
        if (c == '{') {
            v.kind = Json::Object;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == '}') {
                ++i_;
                return v;
            }
            for (;;) {
                ws();
                std::string key = string_lit();
                ws();
                if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
                ++i_;
                v.fields.emplace_back(std::move(key), value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == '}') {
                    ++i_;
                    return v;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = Json::Array;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == ']') {
                ++i_;
                return v;
            }
            for (;;) {
                v.items.push_back(value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == ']') {
                    ++i_;
                    return v;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = Json::String;
            v.text = string_lit();
            return v;
        }
        if (s_.compare(i_, 4, "true") == 0) {
            i_ += 4;
            v.kind = Json::Bool;
            v.b = true;
            return v;
        }
        if (s_.compare(i_, 5, "false") == 0) {
            i_ += 5;
            v.kind = Json::Bool;
            return v;
        }
        if (s_.compare(i_, 4, "null") == 0) {
            i_ += 4;
            return v;
        }
        const size_t b = i_;
        while (i_ < s_.size() && (std::strchr("+-0123456789.eE", s_[i_]) != nullptr)) ++i_;
        if (i_ == b) fail("unexpected character");
        v.kind = Json::Number;
        v.text = s_.substr(b, i_ - b);
        return v;
    }
    std::string string_lit() {
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected a string");
        ++i_;
        std::string out;
        while (i_ < s_.size() && s_[i_] != '"') {
            char c = s_[i_++];
            if (c == '\\') {
                if (i_ >= s_.size()) fail("bad escape");
                const char e = s_[i_++];
                switch (e) {
                    case '"': c = '"'; break;
                    case '\\': c = '\\'; break;
                    case '/': c = '/'; break;
                    case 'b': c = '\b'; break;
                    case 'f': c = '\f'; break;
                    case 'n': c = '\n'; break;
                    case 'r': c = '\r'; break;
                    case 't': c = '\t'; break;
                    case 'u': {  // layer names are ASCII; keep BMP code points < 0x80 only
                        if (i_ + 4 > s_.size()) fail("bad \\u escape");
                        const long cp = std::strtol(s_.substr(i_, 4).c_str(), nullptr, 16);
                        i_ += 4;
                        if (cp >= 0x80) fail("non-ASCII \\u escape");
                        c = static_cast<char>(cp);
                        break;
                    }
                    default: fail("bad escape");
                }
            }
            out.push_back(c);
        }
        if (i_ >= s_.size()) fail("unterminated string");
        ++i_;
        return out;
    }
    const std::string& s_;
    size_t i_ = 0;
};

std::string load_text(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(FQG_ERR_RUNTIME, "cannot open " + path);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

// schemas.cpp:20-27 parse_real: the whole literal must be consumed.
double parse_real(const std::string& text) {
    char* end = nullptr;
    const double v = std::strtod(text.c_str(), &end);
    if (end == text.c_str() || *end != '\0') throw Error(FQG_ERR_INVALID, "bad real literal: " + text);
    return v;
}

// ------------------------------------------------------------------ FQTA
struct Tensor {
    std::string name;
    bool is_f64 = true;
    int64_t rows = 0, cols = 0;
    std::vector<double> f;
    std::vector<int32_t> i;
};

constexpr uint64_t kMaxElements = uint64_t{1} << 36;  // archive.cpp:16

std::vector<Tensor> read_fqta(const std::string& path) {
    const std::string bytes = load_text(path);
    size_t pos = 0;
    auto take = [&](size_t n) -> const char* {
        if (bytes.size() - pos < n) throw Error(FQG_ERR_RUNTIME, "truncated payload");
        const char* p = bytes.data() + pos;
        pos += n;
        return p;
    };
    auto u32 = [&] {
        uint32_t v;
        std::memcpy(&v, take(4), 4);  // little-endian host (x86-64 / aarch64)
        return v;
    };
    auto u64 = [&] {
        uint64_t v;
        std::memcpy(&v, take(8), 8);
        return v;
    };
    if (std::memcmp(take(4), "FQTA", 4) != 0) throw Error(FQG_ERR_RUNTIME, "bad magic (not an FQTA file)");
    const uint32_t version = u32();
    if (version != 1) throw Error(FQG_ERR_RUNTIME, "unsupported version " + std::to_string(version));
    const uint32_t count = u32();
    std::vector<Tensor> out;
    std::unordered_set<std::string> seen;
    for (uint32_t t = 0; t < count; ++t) {
        Tensor x;
        const uint32_t nl = u32();
        x.name.assign(take(nl), nl);
        if (!seen.insert(x.name).second) throw Error(FQG_ERR_RUNTIME, "duplicate tensor name: " + x.name);
        const uint8_t dtype = static_cast<uint8_t>(*take(1));
        if (dtype != 0 && dtype != 1)
            throw Error(FQG_ERR_RUNTIME, "unknown dtype tag " + std::to_string(dtype));
        const uint32_t ndim = u32();
        if (ndim != 2) throw Error(FQG_ERR_RUNTIME, "unsupported ndim " + std::to_string(ndim) + " (expected 2)");
        const uint64_t rows = u64(), cols = u64();
        if (rows < 1 || cols < 1 || rows > kMaxElements || cols > kMaxElements || rows * cols > kMaxElements)
            throw Error(FQG_ERR_RUNTIME, "invalid tensor dims");
        x.rows = static_cast<int64_t>(rows);
        x.cols = static_cast<int64_t>(cols);
        const size_t n = static_cast<size_t>(rows * cols);
        if (dtype == 0) {
            const char* src = take(n * 8);  // bounds-checked before the allocation
            x.f.resize(n);
            std::memcpy(x.f.data(), src, n * 8);
            for (double v : x.f)
                if (!std::isfinite(v)) throw Error(FQG_ERR_RUNTIME, "non-finite value in tensor: " + x.name);
        } else {
            x.is_f64 = false;
            const char* src = take(n * 4);
            x.i.resize(n);
            std::memcpy(x.i.data(), src, n * 4);
        }
        out.push_back(std::move(x));
    }
    if (pos != bytes.size()) throw Error(FQG_ERR_RUNTIME, "trailing bytes after last tensor");
    return out;
}

// archive.cpp:94-120 encode_archive for f64 tensors.
void write_fqta_f64(const std::string& path, const std::vector<Tensor>& ts) {
    std::string out = "FQTA";
    auto put = [&out](const void* p, size_t n) { out.append(static_cast<const char*>(p), n); };
    const uint32_t version = 1, count = static_cast<uint32_t>(ts.size()), two = 2;
    put(&version, 4);
    put(&count, 4);
    for (const Tensor& t : ts) {
        const uint32_t nl = static_cast<uint32_t>(t.name.size());
        put(&nl, 4);
        put(t.name.data(), nl);
        out.push_back('\0');  // kDtypeF64
        put(&two, 4);
        const uint64_t r = static_cast<uint64_t>(t.rows), c = static_cast<uint64_t>(t.cols);
        put(&r, 8);
        put(&c, 8);
        put(t.f.data(), t.f.size() * 8);
    }
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw Error(FQG_ERR_RUNTIME, "cannot open " + path + " for writing");
    f.write(out.data(), static_cast<std::streamsize>(out.size()));
    if (!f) throw Error(FQG_ERR_RUNTIME, "write failed: " + path);
}

// ------------------------------------------------------------------ recipe
struct PlanRec {
    double t = 0;
    int64_t block = 32, padded = 0;
    std::vector<int64_t> e;
};

// schemas.cpp:80-96 plan_from_json, with its consistency checks.
PlanRec plan_from_json(const Json& j) {
    PlanRec p;
    p.t = j.at("T").num();
    for (const Json& v : j.at("E").items) {
        const int64_t e = v.integer();
        if (e < 0) throw Error(FQG_ERR_INVALID, "plan: negative extension count");
        p.e.push_back(e);
    }
    p.block = j.at("block").integer();
    int64_t c_extend = 0;
    for (int64_t e : p.e) c_extend += e;
    p.padded = j.at("padded_width").integer();
    const int64_t width = static_cast<int64_t>(p.e.size()) + c_extend;
    if (p.block < 1 || c_extend != j.at("c_extend").integer() ||
        p.padded != (width + p.block - 1) / p.block * p.block)
        throw Error(FQG_ERR_INVALID, "plan: inconsistent extension counts");
    return p;
}

struct LayerRec {
    std::string name, mode;
    int bits = 8;
    std::vector<double> s;
    PlanRec px, pw;
    double act_scale = 0, w_scale = 0, kl_act = 0, kl_w = 0;
    std::vector<int32_t> wq;  // [K'][N] from "<layer>.qweight"
    int64_t n = 0;
};

}  // namespace
}  // namespace fqg

struct fqg_model_s {
    std::vector<fqg::LayerRec> recs;
    std::vector<fqg_layer_t> layers;  // null when loaded with device < 0 (parse only)
    ~fqg_model_s() {
        for (fqg_layer_t l : layers)
            if (l) fqg_layer_destroy(l);
    }
};

using namespace fqg;

extern "C" {

int fqg_model_load(const char* recipe_path, const char* qmodel_path, int device, int a_format,
                   fqg_model_t* out) {
    return guard([&] {
        require(recipe_path && out, "fqg_model_load: null argument");
        const std::string text = load_text(recipe_path);
        const Json j = JsonParser(text).parse();
        const int64_t version = j.at("schema_version").integer();
        if (version != 1)  // schemas.cpp:166-172 check_version
            throw Error(FQG_ERR_INVALID, "unsupported schema_version " + std::to_string(version));
        std::unique_ptr<fqg_model_s> m(new fqg_model_s());
        for (const Json& l : j.at("layers").items) {  // schemas.cpp:268-295 parse_recipe_json
            LayerRec r;
            r.name = l.at("layer").str();
            r.mode = l.at("mode").str();
            r.bits = static_cast<int>(l.at("bits").integer());
            if (r.bits != 4 && r.bits != 8) throw Error(FQG_ERR_INVALID, "recipe: bits must be 4 or 8");
            for (const Json& v : l.at("smooth_scales").items) r.s.push_back(parse_real(v.str()));
            r.px = plan_from_json(l.at("plan_x"));
            r.pw = plan_from_json(l.at("plan_w"));
            r.act_scale = parse_real(l.at("act_scale").str());
            r.w_scale = parse_real(l.at("weight_scale").str());
            r.kl_act = l.at("kl_ratio_act").num();
            r.kl_w = l.at("kl_ratio_w").num();
            require(static_cast<int64_t>(r.s.size()) == static_cast<int64_t>(r.px.e.size()),
                    "recipe: smoothing scales do not match plan_x");
            require(static_cast<int64_t>(r.pw.e.size()) == r.px.padded,
                    "recipe: plan_w does not match plan_x's padded width");
            m->recs.push_back(std::move(r));
        }
        if (qmodel_path != nullptr) {  // flattenquant_cli.cpp:247-249 qmodel.require(...).int_matrix()
            std::vector<Tensor> ts = read_fqta(qmodel_path);
            for (LayerRec& r : m->recs) {
                const std::string want = r.name + ".qweight";
                Tensor* t = nullptr;
                for (Tensor& x : ts)
                    if (x.name == want) t = &x;
                if (t == nullptr) throw Error(FQG_ERR_RUNTIME, "missing tensor: " + want);
                if (t->is_f64) throw Error(FQG_ERR_RUNTIME, "tensor " + want + " is not int32");
                require(t->rows == r.pw.padded, "recipe: weight_q rows do not match plan_w");
                r.n = t->cols;
                r.wq = std::move(t->i);
            }
        }
        if (device >= 0) {
            require(qmodel_path != nullptr, "fqg_model_load: the quantized archive is required");
            for (const LayerRec& r : m->recs) {
                fqg_layer_desc d{};
                d.bits = r.bits;
                d.k = static_cast<int64_t>(r.s.size());
                d.n = r.n;
                d.smooth_scales = r.s.data();
                d.t_x = r.px.t;
                d.ext_x = r.px.e.data();
                d.block_x = r.px.block;
                d.t_w = r.pw.t;
                d.ext_w = r.pw.e.data();
                d.block_w = r.pw.block;
                d.act_scale = r.act_scale;
                d.weight_q = r.wq.data();
                d.w_scale = r.w_scale;
                d.n_total = r.n;
                d.a_format = r.bits == 4 ? a_format : FQG_I8;
                d.b_format = r.bits == 4 ? FQG_I4 : FQG_I8;
                d.scale_mode = FQG_SCALE_STATIC;
                d.device = device;
                fqg_layer_t h = nullptr;
                const int rc = fqg_layer_create(&d, &h);
                if (rc != FQG_OK) throw Error(rc, r.name + ": " + g_last_error);
                m->layers.push_back(h);
            }
        }
        *out = m.release();
    });
}

int fqg_model_destroy(fqg_model_t m) {
    return guard([&] { delete m; });
}

int fqg_model_num_layers(fqg_model_t m, int64_t* n) {
    return guard([&] {
        require(m && n, "fqg_model_num_layers: null argument");
        *n = static_cast<int64_t>(m->recs.size());
    });
}

int fqg_model_layer_name(fqg_model_t m, int64_t i, char* buf, int64_t cap) {
    return guard([&] {
        require(m && buf && i >= 0 && i < static_cast<int64_t>(m->recs.size()),
                "fqg_model_layer_name: bad argument");
        const std::string& s = m->recs[i].name;
        require(cap > static_cast<int64_t>(s.size()), "fqg_model_layer_name: buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

int fqg_model_layer_recipe(fqg_model_t m, int64_t i, fqg_layer_desc* d, double* kl_ratio_act,
                           double* kl_ratio_w) {
    return guard([&] {
        require(m && d && i >= 0 && i < static_cast<int64_t>(m->recs.size()),
                "fqg_model_layer_recipe: bad argument");
        const LayerRec& r = m->recs[i];
        *d = fqg_layer_desc{};
        d->bits = r.bits;
        d->k = static_cast<int64_t>(r.s.size());
        d->n = r.n;
        d->smooth_scales = r.s.data();
        d->t_x = r.px.t;
        d->ext_x = r.px.e.data();
        d->block_x = r.px.block;
        d->t_w = r.pw.t;
        d->ext_w = r.pw.e.data();
        d->block_w = r.pw.block;
        d->act_scale = r.act_scale;
        d->weight_q = r.wq.empty() ? nullptr : r.wq.data();
        d->w_scale = r.w_scale;
        d->n_total = r.n;
        if (kl_ratio_act) *kl_ratio_act = r.kl_act;
        if (kl_ratio_w) *kl_ratio_w = r.kl_w;
    });
}

int fqg_model_layer(fqg_model_t m, const char* name, fqg_layer_t* layer) {
    return guard([&] {
        require(m && name && layer, "fqg_model_layer: null argument");
        require(!m->layers.empty(), "fqg_model_layer: model was loaded without a device");
        for (size_t i = 0; i < m->recs.size(); ++i)
            if (m->recs[i].name == name) {
                *layer = m->layers[i];
                return;
            }
        throw Error(FQG_ERR_RUNTIME, std::string("no recipe for ") + name);
    });
}

int fqg_model_infer(fqg_model_t m, const char* input_path, const char* out_path,
                    int64_t* saturated_total, int64_t* ran) {
    return guard([&] {
        require(m && input_path && out_path, "fqg_model_infer: null argument");
        require(!m->layers.empty(), "fqg_model_infer: model was loaded without a device");
        std::vector<Tensor> inputs = read_fqta(input_path);
        std::vector<Tensor> outputs;
        int64_t sat_total = 0, count = 0;
        for (const Tensor& in : inputs) {  // flattenquant_cli.cpp:261-273
            const auto slash = in.name.find('/');
            if (slash == std::string::npos || !in.is_f64) continue;
            const std::string layer = in.name.substr(0, slash);
            fqg_layer_t h = nullptr;
            size_t li = 0;
            for (; li < m->recs.size(); ++li)
                if (m->recs[li].name == layer) {
                    h = m->layers[li];
                    break;
                }
            if (h == nullptr) throw Error(FQG_ERR_RUNTIME, "no recipe for " + layer);
            if (in.cols != static_cast<int64_t>(m->recs[li].s.size()))  // pipeline.cpp:161-163
                throw Error(FQG_ERR_INVALID, "run_layer: input channel count does not match recipe");
            Tensor o;
            o.name = in.name;
            o.rows = in.rows;
            o.cols = m->recs[li].n;
            o.f.resize(static_cast<size_t>(o.rows * o.cols));
            int64_t sat = 0;
            const int rc = fqg_layer_run_host(h, in.f.data(), in.rows, o.f.data(), &sat);
            if (rc != FQG_OK) throw Error(rc, g_last_error);
            sat_total += sat;
            ++count;
            outputs.push_back(std::move(o));
        }
        if (count == 0) throw Error(FQG_ERR_RUNTIME, "input archive has no <layer>/<name> tensors");
        write_fqta_f64(out_path, outputs);
        if (saturated_total) *saturated_total = sat_total;
        if (ran) *ran = count;
    });
}

}  // extern "C"
