// mcx/json_lite.hpp -- the small JSON subset the encoder sidecar and table
// schemas use (dataset.hpp:83-463 reads and writes them with nlohmann::json,
// a dependency this drop-in does not take): null, booleans, numbers
// (integers kept exact up to 64 bits), strings with the standard escapes,
// arrays and objects.  Objects keep their keys sorted, as nlohmann::json's
// default std::map does, so dumps list keys in the same order.
#pragma once

#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace mcx::json {

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Value {
public:
    enum class Type { null, boolean, number, string, array, object };

    Value() = default;
    Value(std::nullptr_t) {}
    Value(bool b) : type_(Type::boolean), b_(b) {}
    Value(double d) : type_(Type::number), d_(d) {}
    Value(int v) : Value(static_cast<std::int64_t>(v)) {}
    Value(unsigned v) : Value(static_cast<std::uint64_t>(v)) {}
    Value(std::int64_t v) : type_(Type::number), d_(double(v)), integral_(true), neg_(v < 0), u_(std::uint64_t(v)) {}
    Value(std::uint64_t v) : type_(Type::number), d_(double(v)), integral_(true), neg_(false), u_(v) {}
    Value(const char* s) : type_(Type::string), s_(s) {}
    Value(std::string s) : type_(Type::string), s_(std::move(s)) {}
    Value(const std::vector<std::string>& v) : type_(Type::array) {
        for (const auto& s : v) a_.emplace_back(s);
    }
    static Value array() {
        Value v;
        v.type_ = Type::array;
        return v;
    }
    static Value object() {
        Value v;
        v.type_ = Type::object;
        return v;
    }

    Type type() const noexcept { return type_; }
    bool is_array() const noexcept { return type_ == Type::array; }
    bool is_object() const noexcept { return type_ == Type::object; }
    bool contains(const std::string& k) const { return type_ == Type::object && o_.count(k); }
    bool empty() const noexcept { return type_ == Type::array ? a_.empty() : type_ == Type::object ? o_.empty() : true; }

    const Value& at(const std::string& k) const {
        if (type_ != Type::object) throw ParseError("not an object");
        const auto it = o_.find(k);
        if (it == o_.end()) throw ParseError("key '" + k + "' not found");
        return it->second;
    }
    Value& operator[](const std::string& k) {
        if (type_ == Type::null) type_ = Type::object;
        if (type_ != Type::object) throw ParseError("not an object");
        return o_[k];
    }
    void push_back(Value v) {
        if (type_ == Type::null) type_ = Type::array;
        if (type_ != Type::array) throw ParseError("not an array");
        a_.push_back(std::move(v));
    }
    const std::vector<Value>& items() const {
        if (type_ != Type::array) throw ParseError("not an array");
        return a_;
    }

    std::string str() const {
        if (type_ != Type::string) throw ParseError("type must be string");
        return s_;
    }
    bool boolean() const {
        if (type_ != Type::boolean) throw ParseError("type must be boolean");
        return b_;
    }
    double number() const {
        if (type_ != Type::number) throw ParseError("type must be number");
        return d_;
    }
    std::uint64_t u64() const {
        if (type_ != Type::number || !integral_ || neg_) throw ParseError("type must be an unsigned integer");
        return u_;
    }
    std::int64_t i64() const {
        if (type_ != Type::number || !integral_) throw ParseError("type must be an integer");
        return static_cast<std::int64_t>(u_);
    }
    std::uint32_t u32() const {
        const std::uint64_t v = u64();
        if (v > 0xffffffffull) throw ParseError("value out of range");
        return std::uint32_t(v);
    }
    std::vector<std::string> strings() const {
        std::vector<std::string> out;
        for (const auto& v : items()) out.push_back(v.str());
        return out;
    }
    // value(key, default) for objects
    template <class T>
    T get_or(const std::string& k, T dflt) const;

    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }

    static Value parse(const std::string& text) {
        std::size_t pos = 0;
        Value v = parse_value(text, pos);
        skip_ws(text, pos);
        if (pos != text.size()) throw ParseError("syntax error at byte " + std::to_string(pos) + ": trailing data");
        return v;
    }

private:
    static void skip_ws(const std::string& t, std::size_t& p) {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
    }
    [[noreturn]] static void fail(std::size_t p, const char* what) {
        throw ParseError("syntax error at byte " + std::to_string(p) + ": " + what);
    }
    static std::string parse_string(const std::string& t, std::size_t& p) {
        if (t[p] != '"') fail(p, "expected string");
        ++p;
        std::string s;
        while (p < t.size() && t[p] != '"') {
            char c = t[p++];
            if (c != '\\') {
                s.push_back(c);
                continue;
            }
            if (p >= t.size()) fail(p, "bad escape");
            c = t[p++];
            switch (c) {
                case '"': s.push_back('"'); break;
                case '\\': s.push_back('\\'); break;
                case '/': s.push_back('/'); break;
                case 'b': s.push_back('\b'); break;
                case 'f': s.push_back('\f'); break;
                case 'n': s.push_back('\n'); break;
                case 'r': s.push_back('\r'); break;
                case 't': s.push_back('\t'); break;
                case 'u': {
                    if (p + 4 > t.size()) fail(p, "bad \\u escape");
                    const unsigned cp = unsigned(std::stoul(t.substr(p, 4), nullptr, 16));
                    p += 4;
                    if (cp < 0x80) s.push_back(char(cp));
                    else if (cp < 0x800) {
                        s.push_back(char(0xc0 | (cp >> 6)));
                        s.push_back(char(0x80 | (cp & 0x3f)));
                    } else {
                        s.push_back(char(0xe0 | (cp >> 12)));
                        s.push_back(char(0x80 | ((cp >> 6) & 0x3f)));
                        s.push_back(char(0x80 | (cp & 0x3f)));
                    }
                    break;
                }
                default: fail(p, "bad escape");
            }
        }
        if (p >= t.size()) fail(p, "unterminated string");
        ++p;
        return s;
    }
    static Value parse_value(const std::string& t, std::size_t& p) {
        skip_ws(t, p);
        if (p >= t.size()) fail(p, "unexpected end of input");
        const char c = t[p];
        if (c == '{') {
            Value v = object();
            ++p;
            skip_ws(t, p);
            if (p < t.size() && t[p] == '}') return ++p, v;
            for (;;) {
                skip_ws(t, p);
                std::string k = parse_string(t, p);
                skip_ws(t, p);
                if (p >= t.size() || t[p] != ':') fail(p, "expected ':'");
                ++p;
                v.o_[k] = parse_value(t, p);
                skip_ws(t, p);
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == '}') return ++p, v;
                fail(p, "expected ',' or '}'");
            }
        }
        if (c == '[') {
            Value v = array();
            ++p;
            skip_ws(t, p);
            if (p < t.size() && t[p] == ']') return ++p, v;
            for (;;) {
                v.a_.push_back(parse_value(t, p));
                skip_ws(t, p);
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == ']') return ++p, v;
                fail(p, "expected ',' or ']'");
            }
        }
        if (c == '"') return Value(parse_string(t, p));
        if (t.compare(p, 4, "true") == 0) return p += 4, Value(true);
        if (t.compare(p, 5, "false") == 0) return p += 5, Value(false);
        if (t.compare(p, 4, "null") == 0) return p += 4, Value();
        // number: integers exact in 64 bits, everything else as double
        const std::size_t b = p;
        if (t[p] == '-') ++p;
        bool frac = false;
        while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '.' || t[p] == 'e' ||
                                t[p] == 'E' || t[p] == '+' || t[p] == '-')) {
            if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') frac = true;
            ++p;
        }
        const std::string num = t.substr(b, p - b);
        if (num.empty() || num == "-") fail(b, "invalid literal");
        try {
            if (!frac) {
                if (num[0] == '-') return Value(static_cast<std::int64_t>(std::stoll(num)));
                return Value(static_cast<std::uint64_t>(std::stoull(num)));
            }
            return Value(std::stod(num));
        } catch (const std::exception&) {
            fail(b, "invalid number");
        }
    }
    static void write_string(std::string& out, const std::string& s) {
        out.push_back('"');
        for (const char c : s) {
            switch (c) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\n': out += "\\n"; break;
                case '\r': out += "\\r"; break;
                case '\t': out += "\\t"; break;
                case '\b': out += "\\b"; break;
                case '\f': out += "\\f"; break;
                default:
                    if (static_cast<unsigned char>(c) < 0x20) {
                        char buf[8];
                        std::snprintf(buf, sizeof(buf), "\\u%04x", unsigned(c));
                        out += buf;
                    } else {
                        out.push_back(c);
                    }
            }
        }
        out.push_back('"');
    }
    void write(std::string& out, int indent, int depth) const {
        auto nl = [&](int d) {
            if (indent < 0) return;
            out.push_back('\n');
            out.append(std::size_t(indent) * std::size_t(d), ' ');
        };
        switch (type_) {
            case Type::null: out += "null"; break;
            case Type::boolean: out += b_ ? "true" : "false"; break;
            case Type::number: {
                if (integral_) {
                    out += neg_ ? std::to_string(static_cast<std::int64_t>(u_)) : std::to_string(u_);
                } else {
                    char buf[40];
                    std::snprintf(buf, sizeof(buf), "%.17g", d_);  // round-trips exactly
                    std::string s = buf;
                    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
                    out += s;
                }
                break;
            }
            case Type::string: write_string(out, s_); break;
            case Type::array: {
                out.push_back('[');
                for (std::size_t i = 0; i < a_.size(); ++i) {
                    if (i) out.push_back(',');
                    nl(depth + 1);
                    a_[i].write(out, indent, depth + 1);
                }
                if (!a_.empty()) nl(depth);
                out.push_back(']');
                break;
            }
            case Type::object: {
                out.push_back('{');
                std::size_t i = 0;
                for (const auto& [k, v] : o_) {
                    if (i++) out.push_back(',');
                    nl(depth + 1);
                    write_string(out, k);
                    out += indent < 0 ? ":" : ": ";
                    v.write(out, indent, depth + 1);
                }
                if (!o_.empty()) nl(depth);
                out.push_back('}');
                break;
            }
        }
    }

    Type type_ = Type::null;
    bool b_ = false;
    double d_ = 0;
    bool integral_ = false, neg_ = false;
    std::uint64_t u_ = 0;
    std::string s_;
    std::vector<Value> a_;
    std::map<std::string, Value> o_;
};

template <>
inline std::string Value::get_or<std::string>(const std::string& k, std::string d) const {
    return contains(k) ? at(k).str() : d;
}
template <>
inline std::uint32_t Value::get_or<std::uint32_t>(const std::string& k, std::uint32_t d) const {
    return contains(k) ? at(k).u32() : d;
}

}  // namespace mcx::json
