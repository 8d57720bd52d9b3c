# Structural oracle: build the reference library (stagekit, /root/reference/proj) out of tree
# into oracle/_ref/.  Never copies reference sources into the repo: every object is compiled
# from the file where it lies under /root/reference; the one source that does not compile as
# shipped (proj/src/codegen.cpp: `using minic::Expr;` clashes with stagekit::Expr)
# is sed-patched into oracle/_ref/ at build time (git-ignored, never committed).  The vendored
# JSON header the reference expects (proj/.gitignore:2) comes from the image's cudnn_frontend.
REF      ?= /root/reference/proj
OUT      := _ref
JSON_HPP ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp
CXX      ?= g++
CXXFLAGS ?= -std=c++20 -O2 -fPIC -w -I$(REF)/include -I$(OUT)/vendor
TUS      := expr graph stage records loops vectordsl schedule fusion dump minic
OBJS     := $(addprefix $(OUT)/,$(addsuffix .o,$(TUS))) $(OUT)/codegen.o

all: $(OUT)/libstagekit.a $(OUT)/stage_programs $(OUT)/run_staged

$(OUT)/vendor/json.hpp:
	@mkdir -p $(OUT)/vendor
	cp $(JSON_HPP) $@

$(OUT)/%.o: $(REF)/src/%.cpp $(OUT)/vendor/json.hpp
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/codegen_patched.cpp: $(REF)/src/codegen.cpp
	@mkdir -p $(OUT)
	sed -e 's/^using minic::Expr;/namespace mc = minic;/' \
	    -e 's/\bExpr::\(int_lit\|double_lit\|bool_lit\|str_lit\|unit\|ref\|unary\|binary\|call\|index\|cond\|K\)\b/mc::Expr::\1/g' \
	    -e 's/std::make_shared<Expr>/std::make_shared<mc::Expr>/g' $< > $@

$(OUT)/codegen.o: $(OUT)/codegen_patched.cpp $(OUT)/vendor/json.hpp
	$(CXX) $(CXXFLAGS) -I$(REF)/src -c $< -o $@

$(OUT)/libstagekit.a: $(OBJS)
	ar rcs $@ $^

# stage_programs: stages the hot-path programs through the reference DSL (fuse_loops with
# motion off, build_schedule, run_codegen) and writes the staged fixtures under
# tests/golden/staged/ (integration/stage_programs.cpp + the serializer
# integration/stagekit_dlx.cpp + the MiniC evaluator oracle/minic_eval.hpp: our code).
$(OUT)/stage_programs: ../integration/stage_programs.cpp ../integration/stagekit_dlx.cpp \
                      ../integration/stagekit_dlx.hpp minic_eval.hpp $(OUT)/libstagekit.a
	$(CXX) $(CXXFLAGS) -I.. -o $@ ../integration/stage_programs.cpp ../integration/stagekit_dlx.cpp \
	    $(OUT)/libstagekit.a

# run_staged: the C++ end-to-end drop-in check (reference DSL -> fuse -> schedule ->
# stagekit_dlx::run_on_b200 vs the reference MiniC evaluated on the CPU); links libdlx.so.
DLX_DIR := $(abspath ../paper_1109_0778_b200)
$(OUT)/run_staged: ../integration/run_staged.cpp ../integration/stagekit_dlx.cpp \
                   ../integration/stagekit_dlx_run.cpp ../integration/stagekit_dlx.hpp minic_eval.hpp \
                   $(OUT)/libstagekit.a $(DLX_DIR)/libdlx.so
	$(CXX) $(CXXFLAGS) -I.. -o $@ ../integration/run_staged.cpp ../integration/stagekit_dlx.cpp ../integration/stagekit_dlx_run.cpp \
	    $(OUT)/libstagekit.a -L$(DLX_DIR) -ldlx -Wl,-rpath,'$$ORIGIN/../../paper_1109_0778_b200'

clean:
	rm -rf $(OUT)

.PHONY: all clean
